#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm.py -x -q > gpurun_out/pytest_spmm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmm.log
bash tools/gpu_trace6.sh
TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_base.so timeout 600 python tools/fixed_cost.py > gpurun_out/fixed_base.txt 2>&1
timeout 600 python tools/fixed_cost.py > gpurun_out/fixed_new.txt 2>&1
VARIANTS="base:TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_base.so new:TCSL_X=0" bash tools/gpu_ab2.sh > gpurun_out/ab.txt 2>&1
