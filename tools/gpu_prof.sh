#!/bin/bash
# GPU iteration: parity, quick bench, traces, one ncu --set full capture.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_spmm.py -x -q --timeout 60 > gpurun_out/pytest_spmm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmm.log
CELLS=${CELLS:-ffn1:0.7:16,ffn1:0.8:16,ffn1:0.9:16,out:0.8:16,ffn2:0.9:8,qkv:0.8:64,qkv:0.9:32}
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-cublas --only $CELLS > gpurun_out/quick.json 2> gpurun_out/quick.err
rm -f gpurun_out/trace.txt
for a in "36864 9216 16 0.8" "36864 9216 16 0.9"; do
  timeout 300 python tools/trace_spmm.py $a >> gpurun_out/trace.txt 2>&1
done
PROF=${PROF:-ffn1:0.8:16}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_sm100 -c 1 -f -o gpurun_out/prof python bench.py --steps 1 --warmup 0 --no-graph --no-cublas --no-e2e --no-cpu-baseline --kernel-reps 1 --only $PROF > gpurun_out/ncu_full.log 2>&1
