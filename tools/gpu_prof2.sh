#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/prof_run.txt
for a in "36864 9216 16 0.7" "36864 9216 16 0.9" "36864 9216 16 0.8"; do
  TCSL_DEBUG=16 TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_prof.so timeout 300 python tools/prof_spmm.py $a >> gpurun_out/prof_run.txt 2>&1
done
TCSL_ISSUERS=2 TCSL_DEBUG=16 TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_prof.so timeout 300 python tools/prof_spmm.py 36864 9216 16 0.7 >> gpurun_out/prof_run.txt 2>&1
timeout 600 python tools/c5_shards.py > gpurun_out/c5_shards.json 2> gpurun_out/c5_shards.err
