#!/bin/bash
# Direct aempty waits vs polling-warp release, with 1 or 2 MMA issuers.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_spmm.py -x -q > gpurun_out/pytest_spmm_rel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmm_rel.log
TCSL_ISSUERS=1 timeout 600 python -m pytest tests/test_gpu_spmm.py -x -q > gpurun_out/pytest_spmm_rel1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmm_rel1.log
P=paper_2309_10285_b200/_lib/var_poll.so
VARIANTS="d1:TCSL_ISSUERS=1 d2:TCSL_ISSUERS=2 p1:TCSL_ISSUERS=1,TCSL_CUDA_LIB=$P p2:TCSL_ISSUERS=2,TCSL_CUDA_LIB=$P" bash tools/gpu_ab2.sh > gpurun_out/ab_rel.txt 2>&1
