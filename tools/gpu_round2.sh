#!/bin/bash
# Full GPU session: parity tests, smoke, both bench arms, ncu launch list, ncu --set full
# captures of K2 (three sparsities) and K1, compute-sanitizer runs.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
(nproc; lscpu | head -20) > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
( time timeout 1500 python bench.py ) > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?" >> gpurun_out/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-graph --no-cublas --no-e2e --no-cpu-baseline --kernel-reps 1 --only ffn1:0.8:16,ffn2:0.9:8,qkv:0.7:64,out:0.8:32 > gpurun_out/ncu_launch.log 2>&1
for c in ffn1:0.7:16 ffn1:0.8:16 ffn1:0.9:16; do
  tag=$(echo $c | tr ':.' '__')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_sm100 -c 1 -f -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 0 --no-graph --no-cublas --no-e2e --no-cpu-baseline --kernel-reps 1 --only $c > gpurun_out/ncu_$tag.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"emit128|count128" -c 2 -f -o gpurun_out/prof_enc python tools/time_encode.py 36864 9216 0.8 > gpurun_out/ncu_enc.log 2>&1
bash tools/gpu_sanitize.sh
