#!/bin/bash
mkdir -p gpurun_out
TCSL_ISSUERS=4 timeout 600 python -m pytest tests/test_gpu_spmm.py -x -q > gpurun_out/pytest_spmm_i4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmm_i4.log
CELLS="ffn1:0.9:16,ffn1:0.9:32,out:0.9:8,ffn2:0.9:8,qkv:0.9:64,ffn1:0.8:16,out:0.8:32" VARIANTS="i2:TCSL_X=0 i4:TCSL_ISSUERS=4" bash tools/gpu_ab2.sh > gpurun_out/ab_i4.txt 2>&1
