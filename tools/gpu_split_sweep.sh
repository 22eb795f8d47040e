#!/bin/bash
# Per-cell cold times at forced split-K S = 1..4 and auto, all 84 cells.
mkdir -p gpurun_out
ARGS="--no-e2e --no-cpu-baseline --no-cublas --steps 3 --warmup 3"
for S in 0 1 2 3 4 6; do
  timeout 900 python bench.py $ARGS --split $S > gpurun_out/split_$S.json 2> gpurun_out/split_$S.err
done
