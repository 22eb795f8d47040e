#!/bin/bash
# K1 encoder: parity tests + per-kernel timings on OPT-66B weights.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q > gpurun_out/pytest_enc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_enc.log
: > gpurun_out/time_enc.txt
for a in "36864 9216 0.7" "36864 9216 0.8" "36864 9216 0.9" "9216 9216 0.8" "9216 36864 0.8"; do
  timeout 300 python tools/time_encode.py $a >> gpurun_out/time_enc.txt 2>&1
done
TCSL_ENCODE_SLOW=1 timeout 300 python tools/time_encode.py 36864 9216 0.8 >> gpurun_out/time_enc.txt 2>&1
