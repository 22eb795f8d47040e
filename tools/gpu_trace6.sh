#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/trace6.txt
for a in "256 64 16 0.9" "18944 640 16 0.9" "36864 9216 16 0.9"; do
  echo "=== $a" >> gpurun_out/trace6.txt
  TRACE_START=1 timeout 300 python tools/trace_spmm.py $a 2>&1 | grep -v "^  *[0-9]* |" | grep -v "tile |" >> gpurun_out/trace6.txt
done
