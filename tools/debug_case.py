"""Debug helper: one SpMM case vs the oracle, reporting where the errors are."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2309_10285_b200 as tc  # noqa: E402

if os.environ.get("TCSL_DEBUG_LIB"):  # the -DTCSL_TRACE build: extra device-side checks
    tc.LIB_PATH = os.path.join(tc.LIB_DIR, "libtcsl_cuda_trace.so")

print("imported", flush=True)
P = oracle.port()
m, k, n, beta, seed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
splits = [int(s) for s in sys.argv[6].split(",")] if len(sys.argv) > 6 else [0]
a = P.gen_random_sparse(m, k, beta, seed)
x = P.gen_random_sparse(k, n, 0.0, seed + 1)
dev = torch.device("cuda")
t = tc.encode(torch.from_numpy(a.view(np.int16)).to(dev))
want = P.spmm(P.encode(a), x, 8)
print("oracle done; encoded on GPU", flush=True)
for sp in splits:
    try:
        y = tc.spmm(t, torch.from_numpy(x.view(np.int16)).to(dev), split_k=sp).cpu().numpy()
    except tc.TcslError as e:
        print(f"split={sp}: error {e.status} {e}")
        continue
    err = np.abs(y.astype(np.float64) - want)
    bad = err > 1e-2 * (np.abs(want) + 1)
    rows = np.where(bad.any(1))[0]
    cols = np.where(bad.any(0))[0]
    print(f"split={sp} (auto={tc.auto_split(m, k, n)}): max err {err.max():.3g}, bad {bad.sum()} / {bad.size};"
          f" bad row blocks {sorted(set((rows // 128).tolist()))}, bad cols {cols.tolist()[:20]}")
    if rows.size:
        r = rows[0]
        print("   first bad row", r, "y", y[r, :4], "want", want[r, :4])
