#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/time_cnt.txt
for rep in 1 2; do
for v in base em6 em4; do
  lib=paper_2309_10285_b200/_lib/var_$v.so; [ $v = base ] && lib=paper_2309_10285_b200/_lib/libtcsl_cuda.so
  echo "== $v" >> gpurun_out/time_cnt.txt
  TCSL_CUDA_LIB=$lib timeout 300 python tools/time_encode.py 36864 9216 0.8 >> gpurun_out/time_cnt.txt 2>&1
done
done
