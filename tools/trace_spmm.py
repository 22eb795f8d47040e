"""Debug-only: per-role clock64 timeline of CTA 0 of the SpMM kernel.

Builds with -DTCSL_TRACE into _lib/libtcsl_cuda_trace.so (never used by the
product path), runs one SpMM and prints where the cycles go per k-tile."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_10285_b200 as tc  # noqa: E402

tc.LIB_PATH = os.path.join(tc.LIB_DIR, "libtcsl_cuda_trace.so")
L = tc.lib()
L.tcsl_cuda_debug_set_trace.argtypes = [C.c_void_p]

M, K, N, beta = [float(v) if i == 3 else int(v) for i, v in enumerate(sys.argv[1:5])] if len(sys.argv) > 4 else (36864, 9216, 16, 0.8)
split = int(sys.argv[5]) if len(sys.argv) > 5 else 0
w = tc.gen_synthetic(M, K, beta, 1)
x = tc.gen_synthetic(K, N, 0.0, 2)
t = tc.encode(w)
del w
y = tc.spmm(t, x, split_k=split)
trace = torch.zeros(13 * 4096, dtype=torch.int64, device="cuda")
L.tcsl_cuda_debug_set_trace(C.c_void_p(trace.data_ptr()))
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
y = tc.spmm(t, x, split_k=split)
e.record()
torch.cuda.synchronize()
print(f"M={M} K={K} N={N} beta={beta} split={tc.auto_split(M, K, N) if not split else split}: {s.elapsed_time(e)*1e3:.1f} us (traced)")
tr = trace.view(13, 4096).cpu().numpy().astype(np.int64)
n = int((tr[5] > 0).sum())
ch = int((tr[9] > 0).sum())
t0 = tr[5][0]
def st(name, v):
    v = v[v != 0] if v.ndim else v
    print(f"  {name:38s} mean {np.mean(v):9.1f}  p50 {np.median(v):9.1f}  p90 {np.percentile(v, 90):9.1f}")
d = slice(2, n - 2)
st("decode: wait aempty (s1-s0)", (tr[1] - tr[0])[d])
st("decode: memset+barrier (s2-s1)", (tr[2] - tr[1])[d])
st("decode: groups (s3-s2)", (tr[3] - tr[2])[d])
st("decode: fence+arrive (s4-s3)", (tr[4] - tr[3])[d])
st("decode: team tile period (s0[i+2]-s0[i])", (tr[0][2:n] - tr[0][:n - 2])[2:-2])
st("mma: wait afull (s6-s5)", (tr[6] - tr[5])[d])
st("mma: wait xfull (s7-s6)", (tr[7] - tr[6])[d])
st("mma: issue->complete (s8-s7)", (tr[8] - tr[7])[d])
st("mma: tile period (s5[i+1]-s5[i])", np.diff(tr[5][:n])[2:-2])
st("decode done -> mma sees afull (s6-s4)", (tr[6] - tr[4])[d])
st("producer: wait eempty (s10-s9)", (tr[10] - tr[9])[2:ch - 2])
st("producer: chunk period", np.diff(tr[9][:ch])[2:-2])
print(f"  tiles traced {n}, chunks {ch}, total cycles {tr[8][n-1]-t0}")
st("decode w0: cycles in chunk waits per tile", tr[11][d])
st("decode w0: chunk waits per tile", tr[12][d].astype(float))
