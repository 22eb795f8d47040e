#!/bin/bash
# GPU iteration: SpMM parity tests first (bounded), then a bench subset.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_spmm.py -x -q > gpurun_out/pytest_spmm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmm.log
CELLS=${CELLS:-ffn1:0.7:16,ffn1:0.8:16,ffn1:0.9:16,out:0.8:16,ffn2:0.9:8,qkv:0.8:64,qkv:0.9:32}
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-cublas --only $CELLS > gpurun_out/quick.json 2> gpurun_out/quick.err
