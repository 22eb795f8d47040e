"""One small SpMM per decode-team shape against the oracle, for compute-sanitizer runs.

  compute-sanitizer --tool racecheck python tools/sanitize_case.py
Shapes: 8x2 rescatter (beta 0.95), 8x3 zero fill (0.75), 6x4 rescatter (0.5); N = 16 and 64;
split-K 1 and 2. Small enough that the tool's slowdown stays in seconds."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2309_10285_b200 as tc  # noqa: E402

P = oracle.port()
cases = [(256, 512, n, beta, split) for beta in (0.95, 0.75, 0.5) for n in (16, 64) for split in (1, 2)]
if len(sys.argv) > 1:
    cases = cases[: int(sys.argv[1])]
dev = torch.device("cuda")
bad = 0
for m, k, n, beta, split in cases:
    a = P.gen_random_sparse(m, k, beta, 11)
    x = P.gen_random_sparse(k, n, 0.0, 12)
    t = tc.encode(torch.from_numpy(a.view(np.int16)).to(dev))
    y = tc.spmm(t, torch.from_numpy(x.view(np.int16)).to(dev), split_k=split).cpu().numpy()
    want = P.spmm(P.encode(a), x, 4)
    rel = float(np.linalg.norm(y - want) / max(np.linalg.norm(want), 1e-30))
    ok = rel <= 1e-3
    bad += not ok
    print(f"m={m} k={k} n={n} beta={beta} split={split}: rel_fro={rel:.2e} {'ok' if ok else 'FAIL'}", flush=True)
print("sanitize cases done, failures:", bad)
sys.exit(1 if bad else 0)
