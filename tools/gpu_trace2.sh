#!/bin/bash
# Skeleton traces (TCSL_DEBUG=7: no scatter/clear, no MMA, no ring loads) at beta 0.9.
mkdir -p gpurun_out
: > gpurun_out/trace2.txt
for iss in 1 2; do
  for dbg in 0 7; do
    echo "=== ISSUERS=$iss DBG=$dbg" >> gpurun_out/trace2.txt
    TCSL_DEBUG=$dbg TCSL_ISSUERS=$iss TRACE_DUMP=gpurun_out/tr2_i${iss}_d$dbg.npy timeout 300 python tools/trace_spmm.py 36864 9216 16 0.9 >> gpurun_out/trace2.txt 2>&1
  done
done
