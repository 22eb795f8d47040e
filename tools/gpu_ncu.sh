#!/bin/bash
# One ncu --set full capture (with source) of the SpMM kernel for each cell in $CELLS.
mkdir -p gpurun_out
CELLS=${CELLS:-ffn1:0.9:16,ffn1:0.7:16}
TAG=${TAG:-cur}
n=$(echo $CELLS | tr ',' '\n' | wc -l)
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:spmm_ -c $n -f -o gpurun_out/prof_$TAG \
  python bench.py --only $CELLS --quick --steps 1 --warmup 0 --no-graph > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
