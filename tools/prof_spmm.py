"""Debug-only: cycle accounting of CTA 0's MMA issuer (-DTCSL_TRACE build).

  TCSL_DEBUG=16 python tools/prof_spmm.py M K N beta   (16 = no per-event trace stores)"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_10285_b200 as tc  # noqa: E402

tc.LIB_PATH = os.environ.get("TCSL_CUDA_LIB") or os.path.join(tc.LIB_DIR, "libtcsl_cuda_trace.so")
L = tc.lib()
L.tcsl_cuda_debug_set_trace.argtypes = [C.c_void_p]
M, K, N, beta = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
w = tc.gen_synthetic(M, K, beta, 1)
x = tc.gen_synthetic(K, N, 0.0, 2)
t = tc.encode(w)
del w
tc.spmm(t, x)
trace = torch.zeros(16 * 4096, dtype=torch.int64, device="cuda")
L.tcsl_cuda_debug_set_trace(C.c_void_p(trace.data_ptr()))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
tc.spmm(t, x)
e.record()
torch.cuda.synchronize()
L.tcsl_cuda_debug_set_trace(None)
pr = trace.view(16, 4096)[15].cpu().tolist()
tot = pr[4] or 1
print(f"M={M} K={K} N={N} beta={beta}: {s.elapsed_time(e) * 1e3:.1f} us; MMA warp of CTA 0: total {tot} cycles")
for i, name in [(0, "wait dempty"), (1, "wait xfull"), (2, "wait afull"), (5, "fence+descriptors"),
                (6, "MMA issue"), (7, "commits"), (3, "loop+syncwarp")]:
    print(f"  {name:20s} {pr[i]:10d} cycles  {100.0 * pr[i] / tot:5.1f} %")
tot = pr[15] or 1
print(f"decode warp 0 of CTA 0: total {tot} cycles")
for i, name in enumerate(["meta", "chunk waits", "load+release", "buffer wake", "clear", "team barrier",
                          "scatter+arrive"]):
    print(f"  {name:20s} {pr[8 + i]:10d} cycles  {100.0 * pr[8 + i] / tot:5.1f} %")
