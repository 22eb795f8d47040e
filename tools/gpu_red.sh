#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_epilogue.py tests/test_gpu_push.py -x -q > gpurun_out/pytest_red.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_red.log
CELLS="out:0.9:8,out:0.7:64,qkv:0.8:16,ffn2:0.9:8,ffn1:0.8:16,ffn1:0.7:16,ffn2_175:0.8:32,c1:0.8:16" VARIANTS="new:TCSL_X=0 k3:TCSL_FUSED_SPLITK=0" bash tools/gpu_ab2.sh > gpurun_out/ab.txt 2>&1
