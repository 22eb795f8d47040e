#!/bin/bash
# One ncu --set full capture of K2 per BASELINE config (C1..C4) and K3 at C3.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --no-graph --no-cublas --no-e2e --no-cpu-baseline --kernel-reps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_sm100 -c 1 -f -o gpurun_out/prof_c1 $B --suite c1 --only c1:0.8:16 > gpurun_out/ncu_c1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spmm_sm100|reduce" -c 2 -f -o gpurun_out/prof_c3 $B --only ffn2:0.9:8 > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_sm100 -c 1 -f -o gpurun_out/prof_c4 $B --only ffn1_175:0.8:32 > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_sm100 -c 1 -f -o gpurun_out/prof_out9 $B --only out:0.9:8 > gpurun_out/ncu_out9.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_sm100 -c 1 -f -o gpurun_out/prof_qkv7 $B --only qkv:0.7:64 > gpurun_out/ncu_qkv7.log 2>&1
