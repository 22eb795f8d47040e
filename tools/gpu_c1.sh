B="python bench.py --steps 1 --warmup 0 --no-graph --no-cublas --no-e2e --no-cpu-baseline --kernel-reps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_sm100 -c 1 -f -o gpurun_out/prof_c1 $B --only c1:0.8:16 > gpurun_out/ncu_c1.log 2>&1
timeout 300 python bench.py --only c1:0.8:16,c1:0.7:16,c1:0.9:16 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c1.json 2> gpurun_out/c1.err
