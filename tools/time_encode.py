"""Debug tool: device time of the GPU encoder (K1) on an OPT-66B weight.

  python tools/time_encode.py [M K beta]   (prints ms and GB/s of 2*M*K read + 4E written)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_10285_b200 as tc  # noqa: E402

M, K, beta = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (36864, 9216, 0.8)
w = tc.gen_synthetic(M, K, beta, 1)
t = tc.encode(w)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
s.record()
for _ in range(reps):
    t = tc.encode(w)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
by = 2.0 * M * K + 4.0 * t.n_entries
print(f"encode {M}x{K} beta={beta}: {ms:.3f} ms/encode (host sync for E included), {by / ms / 1e6:.0f} GB/s of 2MK+4E")
