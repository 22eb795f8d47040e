#!/bin/bash
# Cycle accounting (TCSL_PROF build: tools/build_variant.py prof -DTCSL_PROF) with ablations.
# DBGS="0 1 2 4" ARGS="36864 9216 16 0.9" bash tools/gpu_prof_run.sh
mkdir -p gpurun_out
: > gpurun_out/prof_run.txt
for d in ${DBGS:-0}; do
  for a in "${ARGS:-36864 9216 16 0.9}"; do
    echo "TCSL_DEBUG=$d" >> gpurun_out/prof_run.txt
    TCSL_DEBUG=$d TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_${PROFVAR:-prof}.so timeout 300 python tools/prof_spmm.py $a >> gpurun_out/prof_run.txt 2>&1
  done
done
