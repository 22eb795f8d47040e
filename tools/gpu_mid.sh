#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_configs.py -x -q > gpurun_out/pytest_spmm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmm.log
CELLS="ffn1:0.8:16,ffn1:0.8:64,qkv:0.8:8,out:0.8:32,ffn2:0.8:16,ffn1_175:0.8:32,ffn1:0.85:16" VARIANTS="dense3:TCSL_MID=0 mid20:TCSL_MID=1 mid18:TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_kg18.so" bash tools/gpu_ab2.sh > gpurun_out/ab_mid.txt 2>&1
