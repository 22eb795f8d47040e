#!/bin/bash
# A/B of K2 variants on a cell set (per-cell cold timings). VARIANTS: "name:ENV=VAL,ENV=VAL ..."
mkdir -p gpurun_out
CELLS=${CELLS:-ffn1:0.7:16,ffn1:0.8:16,ffn1:0.9:16,out:0.9:8,qkv:0.8:64,ffn2:0.9:8,ffn1_175:0.7:64,qkv:0.7:64}
VARIANTS=${VARIANTS:-"v1:TCSL_K2_V1=1 v2:TCSL_V2OPT=0 v2pf:TCSL_V2OPT=1"}
ARGS="--only $CELLS --no-e2e --no-cpu-baseline --no-cublas --steps 5 --warmup 3"
for rep in 1 2; do
  for v in $VARIANTS; do
    name=${v%%:*}; envs=${v#*:}
    env $(echo $envs | tr ',' ' ') timeout 600 python bench.py $ARGS > gpurun_out/ab_${name}_$rep.json 2> gpurun_out/ab_${name}_$rep.err
  done
done
python - "$VARIANTS" <<'PY'
import json, sys
names = [v.split(":")[0] for v in sys.argv[1].split()]
rows = {}
for tag in names:
    for rep in (1, 2):
        try:
            d = json.load(open(f"gpurun_out/ab_{tag}_{rep}.json"))
        except Exception as e:
            print(tag, rep, "failed", e); continue
        for c in d["cells"]:
            k = (c["shape"], c["sparsity"], c["N"])
            rows.setdefault(k, {}).setdefault(tag, []).append(c["us"])
        print(tag, rep, "value", d["value"], "frac", d["roofline"]["frac"])
for k, v in rows.items():
    print(k, {t: min(x) for t, x in v.items()})
PY
