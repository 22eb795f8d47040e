#!/bin/bash
# Multi-issuer experiment: parity at I=2/4, then A/B of I=1/2/4.
mkdir -p gpurun_out
for i in 2 4; do
  TCSL_ISSUERS=$i timeout 600 python -m pytest tests/test_gpu_spmm.py -x -q > gpurun_out/pytest_spmm_i$i.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmm_i$i.log
done
VARIANTS="i1:TCSL_ISSUERS=1 i2:TCSL_ISSUERS=2 i4:TCSL_ISSUERS=4" bash tools/gpu_ab2.sh > gpurun_out/ab_iss.txt 2>&1
