#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/trace3.txt
for a in "36864 9216 16 0.9" "36864 9216 16 0.7" "9216 9216 8 0.9"; do
  for rep in 1 2; do
  echo "=== $a" >> gpurun_out/trace3.txt
  TRACE_DUMP=gpurun_out/tr3_$(echo $a | tr ' .' '__')_$rep.npy timeout 300 python tools/trace_spmm.py $a >> gpurun_out/trace3.txt 2>&1
  done
done
