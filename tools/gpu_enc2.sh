#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q > gpurun_out/pytest_enc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_enc.log
: > gpurun_out/time_enc.txt
for g in 0; do
  echo "TCSL_EMIT_PER_SM=$g" >> gpurun_out/time_enc.txt
  for a in "36864 9216 0.7" "36864 9216 0.8" "36864 9216 0.9" "9216 9216 0.8"; do
    TCSL_EMIT_PER_SM=$g timeout 300 python tools/time_encode.py $a >> gpurun_out/time_enc.txt 2>&1
  done
done
TCSL_EMIT_PER_SM=${NCU_PER_SM:-0} timeout 600 ncu --set full --import-source on --clock-control none -k regex:emit128 -c 1 -f -o gpurun_out/prof_emit python tools/time_encode.py 36864 9216 0.8 > gpurun_out/ncu_emit.log 2>&1
