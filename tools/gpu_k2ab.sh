#!/bin/bash
# K2 change: SpMM parity tests, A/B against var_base (HEAD's kernel), startup trace.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm.py -x -q > gpurun_out/pytest_spmm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmm.log
VARIANTS=${VARIANTS:-"base:TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_base.so new:TCSL_X=0"} bash tools/gpu_ab2.sh > gpurun_out/ab.txt 2>&1
: > gpurun_out/trace5.txt
for a in "36864 9216 16 0.9" "9216 9216 8 0.9"; do
  echo "=== $a" >> gpurun_out/trace5.txt
  TRACE_START=1 timeout 300 python tools/trace_spmm.py $a 2>&1 | grep -v "^  *[0-9]* |" >> gpurun_out/trace5.txt
done
