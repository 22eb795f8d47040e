#!/bin/bash
# Session-start check: GPU parity tests + a per-cell timing subset of the current kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CELLS=${CELLS:-ffn1:0.7:16,ffn1:0.8:16,ffn1:0.9:16,out:0.9:8,qkv:0.8:64,ffn2:0.9:8,ffn1_175:0.7:64,qkv:0.7:64}
timeout 600 python bench.py --only $CELLS --no-e2e --no-cpu-baseline --no-cublas --steps 5 --warmup 3 > gpurun_out/base.json 2> gpurun_out/base.err
