#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/trace4.txt
for a in "36864 9216 16 0.9" "36864 9216 16 0.7" "9216 9216 8 0.9"; do
  echo "=== $a" >> gpurun_out/trace4.txt
  TRACE_CHAIN=1 TRACE_START=1 TRACE_NA=8 timeout 300 python tools/trace_spmm.py $a >> gpurun_out/trace4.txt 2>&1
done
