"""Debug-only: per-role clock64 timeline of CTA 0 of the SpMM kernel.

Uses the -DTCSL_TRACE build (_lib/libtcsl_cuda_trace.so, never used by the
product path), runs one SpMM and prints where the cycles go per k-tile.
  python tools/trace_spmm.py M K N beta [split]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_10285_b200 as tc  # noqa: E402

tc.LIB_PATH = os.path.join(tc.LIB_DIR, "libtcsl_cuda_trace.so")
if not os.path.exists(tc.LIB_PATH):
    import subprocess
    subprocess.run(["nvcc", *tc.NVCC_FLAGS, "-DTCSL_TRACE", "-o", tc.LIB_PATH,
                    *[os.path.join(tc.CSRC, f) for f in tc.SOURCES]], check=True)
L = tc.lib()
L.tcsl_cuda_debug_set_trace.argtypes = [C.c_void_p]

args = sys.argv[1:]
M, K, N = (int(args[0]), int(args[1]), int(args[2])) if len(args) >= 3 else (36864, 9216, 16)
beta = float(args[3]) if len(args) >= 4 else 0.8
split = int(args[4]) if len(args) >= 5 else 0
w = tc.gen_synthetic(M, K, beta, 1)
x = tc.gen_synthetic(K, N, 0.0, 2)
t = tc.encode(w)
del w
tc.spmm(t, x, split_k=split)
trace = torch.zeros(16 * 4096, dtype=torch.int64, device="cuda")
L.tcsl_cuda_debug_set_trace(C.c_void_p(trace.data_ptr()))
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
tc.spmm(t, x, split_k=split)
e.record()
torch.cuda.synchronize()
L.tcsl_cuda_debug_set_trace(None)
print(f"M={M} K={K} N={N} beta={beta} split={split or tc.auto_split(M, K, N)}: {s.elapsed_time(e) * 1e3:.1f} us")
tr = trace.view(16, 4096).cpu().numpy().astype(np.int64)
n = int((tr[4] > 0).sum())


def st(name, v):
    v = v[np.isfinite(v)]
    if v.size == 0:
        return
    print(f"  {name:40s} mean {np.mean(v):9.1f}  p50 {np.median(v):9.1f}  p90 {np.percentile(v, 90):9.1f}")


def diff(a, b):
    m = (tr[a] != 0) & (tr[b] != 0)
    return (tr[b] - tr[a])[m][2:-2].astype(float)


st("decode: buffer ready -> team barrier passed (s1-s0)", diff(0, 1))
st("decode: barrier -> tile done (s2-s1)", diff(1, 2))
d0 = tr[0][:n][tr[0][:n] != 0]
st("decode: team-tile period (team of tile 0)", np.diff(d0[::3]).astype(float)[1:-1])
st("mma: wait A full (s4-s3)", diff(3, 4))
m3 = tr[3][:n].astype(float)
st("mma: tile period (s3[i+1]-s3[i])", np.diff(m3)[2:-2])
st("decode done -> mma sees it (s4 - s2)", diff(2, 4))
print(f"  tiles traced {n}, total cycles {tr[4][n - 1] - tr[3][0]}")
st("mma: wait X stage (s3 - s8)", diff(8, 3))
base = tr[8][0]
xs = tr[5][tr[5] != 0] - base
ch = tr[6][tr[6] != 0] - base
print("  X stage issue times (cycles from first MMA poll):", xs[:12].tolist())
print("  MMA tile-start times:", (tr[8][:48:4] - base).tolist())
print("  chunk issue times:", ch[:24].tolist())
print("  decode tile-ready times (s0):", (tr[0][:24] - base).tolist())
it = tr[9][tr[9] != 0] - base
print("  poller: pass-1 start", tr[12][0] - base, "loop start", tr[11][0] - base, "iterations traced", it.size)
print("  poller iteration times:", it[:40].tolist())
print("  poller iteration period p50", float(np.median(np.diff(it))) if it.size > 2 else None)
print("  meta publish times (per 32 tiles):", (tr[10][:8] - base).tolist())
# per-tile critical path (team warp 0 of each tile): start, data ready, buffer ready, barrier, done; MMA sees A full
st("decode: start -> data in smem (s14-s13)", diff(13, 14))
st("decode: data -> buffer free (s0-s14)", diff(14, 0))
m = n - 4
prev_done = tr[2][:m]
print("  tile: start, +data, +buf, +bar, +done | mma_afull_seen - done | gap to previous tile's MMA")
for i in range(60, 72):
    print("   %3d: %7d %+6d %+6d %+6d %+6d | %+6d" % (i, tr[13][i] - base, tr[14][i] - tr[13][i], tr[0][i] - tr[14][i],
          tr[1][i] - tr[0][i], tr[2][i] - tr[1][i], tr[4][i] - tr[2][i]))
