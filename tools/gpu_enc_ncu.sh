#!/bin/bash
# K1 emit: grid variants timed, then one ncu --set full capture of the emit kernel.
mkdir -p gpurun_out
: > gpurun_out/time_enc.txt
for g in 0 2 4; do
  echo "TCSL_EMIT_PER_SM=$g" >> gpurun_out/time_enc.txt
  TCSL_EMIT_PER_SM=$g timeout 300 python tools/time_encode.py 36864 9216 0.8 >> gpurun_out/time_enc.txt 2>&1
done
TCSL_EMIT_PER_SM=${NCU_PER_SM:-0} timeout 600 ncu --set full --import-source on --clock-control none -k regex:emit128 -c 1 -f -o gpurun_out/prof_emit python tools/time_encode.py 36864 9216 0.8 > gpurun_out/ncu_emit.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:count128 -c 1 -f -o gpurun_out/prof_count python tools/time_encode.py 36864 9216 0.8 > gpurun_out/ncu_count.log 2>&1
