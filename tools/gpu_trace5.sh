#!/bin/bash
mkdir -p gpurun_out
for a in "36864 9216 16 0.9" "36864 9216 16 0.7"; do
  TRACE_DUMP=gpurun_out/tr5_$(echo $a | tr ' .' '__').npy timeout 300 python tools/trace_spmm.py $a > /dev/null 2>&1
done
