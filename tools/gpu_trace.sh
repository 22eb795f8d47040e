#!/bin/bash
# Per-tile clock64 traces of CTA 0 (TCSL_TRACE build) for a few cells and issuer counts; raw arrays in gpurun_out/.
mkdir -p gpurun_out
: > gpurun_out/trace.txt
for iss in ${ISS:-1 2}; do
  for a in ${SHAPES:-"36864 9216 16 0.9" "36864 9216 16 0.7"}; do
    tag=$(echo "i$iss $a" | tr ' .' '__')
    echo "=== ISSUERS=$iss $a" >> gpurun_out/trace.txt
    TCSL_ISSUERS=$iss TRACE_DUMP=gpurun_out/tr_$tag.npy timeout 300 python tools/trace_spmm.py $a >> gpurun_out/trace.txt 2>&1
  done
done
