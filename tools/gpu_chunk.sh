#!/bin/bash
mkdir -p gpurun_out
TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_ch8.so timeout 900 python -m pytest tests/test_gpu_spmm.py -x -q > gpurun_out/pytest_ch8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ch8.log
VARIANTS="base:TCSL_X=0 ch8:TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_ch8.so ch32:TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_ch32.so" bash tools/gpu_ab2.sh > gpurun_out/ab.txt 2>&1
