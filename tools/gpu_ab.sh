#!/bin/bash
# A/B timing of library variants (tools/build_variant.py), interleaved twice.
# VARS="base grp" CELLS=... bash tools/gpu_ab.sh
mkdir -p gpurun_out
CELLS=${CELLS:-ffn1:0.7:16,ffn1:0.8:16,ffn1:0.9:16,out:0.8:16,ffn2:0.9:8,qkv:0.8:64}
for rep in 1 2; do
  for v in $VARS; do
    TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_$v.so timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e \
      --no-cpu-baseline --no-cublas --only $CELLS > gpurun_out/ab_${v}_$rep.json 2> gpurun_out/ab_${v}_$rep.err
  done
done
python - <<'PY'
import json, os
vs = os.environ["VARS"].split()
rows = {}
for v in vs:
    for rep in (1, 2):
        try:
            d = json.loads(open(f"gpurun_out/ab_{v}_{rep}.json").read().strip().splitlines()[-1])
        except Exception as e:
            print(v, rep, "failed", e); continue
        for c in d["cells"]:
            rows.setdefault(f"{c['shape']}:{c['sparsity']}:{c['N']}", {}).setdefault(v, []).append(c["us"])
with open("gpurun_out/ab.txt", "w") as f:
    for k, r in rows.items():
        line = f"{k:18s} " + "  ".join(f"{v}: {min(r.get(v, [0])):7.1f}us" for v in vs)
        print(line); f.write(line + "\n")
PY
