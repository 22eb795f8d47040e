#!/bin/bash
mkdir -p gpurun_out
TCSL_SPARSE3=1 timeout 900 python -m pytest tests/test_gpu_spmm.py -x -q > gpurun_out/pytest_sparse3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sparse3.log
CELLS="ffn1:0.9:16,ffn1:0.9:64,out:0.9:8,ffn2:0.9:8,qkv:0.9:32,ffn1_175:0.9:32,c1:0.9:16" VARIANTS="s2:TCSL_X=0 s3:TCSL_SPARSE3=1" bash tools/gpu_ab2.sh > gpurun_out/ab.txt 2>&1
