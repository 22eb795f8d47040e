#!/bin/bash
# One full GPU session: parity tests, smoke, bench, ncu launch list + one full capture.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-graph --no-cublas --no-e2e --no-cpu-baseline --kernel-reps 1 --only ffn1:0.8:16,ffn2:0.9:8,qkv:0.7:64,out:0.8:32 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_sm100 -c 1 -f -o gpurun_out/prof python bench.py --steps 1 --warmup 0 --no-graph --no-cublas --no-e2e --no-cpu-baseline --kernel-reps 1 --only ffn1:0.8:16 > gpurun_out/ncu_full.log 2>&1
