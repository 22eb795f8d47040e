#!/bin/bash
# Round-end style bench session: both arms, then the ncu launch list of a short run.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
( time timeout 1500 python bench.py ) > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?" >> gpurun_out/ref.err
if [ -n "$NCU_LAUNCHES" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-graph --quick > gpurun_out/ncu_launch.log 2>&1
fi
