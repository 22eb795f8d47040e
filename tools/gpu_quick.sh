#!/bin/bash
# Quick GPU iteration: a bench subset + per-role traces of CTA 0.
mkdir -p gpurun_out
CELLS=${CELLS:-ffn1:0.7:16,ffn1:0.8:16,ffn1:0.9:16,out:0.8:16,ffn2:0.9:8,qkv:0.8:64}
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-cublas --only $CELLS > gpurun_out/quick.json 2> gpurun_out/quick.err
for a in "36864 9216 16 0.8" "36864 9216 16 0.9" "36864 9216 16 0.7"; do
  timeout 300 python tools/trace_spmm.py $a >> gpurun_out/trace.txt 2>&1
done
