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

tc.LIB_PATH = os.environ.get("TCSL_CUDA_LIB") or os.path.join(tc.LIB_DIR, "libtcsl_cuda_trace.so")
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
trace = torch.zeros(18 * 4096, dtype=torch.int64, device="cuda")
L.tcsl_cuda_debug_set_trace(C.c_void_p(trace.data_ptr()))
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
tc.spmm(t, x, split_k=split)
e.record()
torch.cuda.synchronize()
L.tcsl_cuda_debug_set_trace(None)
print(f"M={M} K={K} N={N} beta={beta} split={split or tc.auto_split(M, K, N)}: {s.elapsed_time(e) * 1e3:.1f} us")
tr = trace.view(18, 4096).cpu().numpy().astype(np.int64)
nb = int((tr[17] > 0).sum())
if nb:
    t0 = tr[16][:nb].min()
    ends = (tr[17][:nb] - t0) / 1e3
    starts = (tr[16][:nb] - t0) / 1e3
    print(f"  CTAs {nb}: start spread {starts.max():.1f} us, end min/median/max {ends.min():.1f} / {np.median(ends):.1f} / {ends.max():.1f} us; slowest CTAs {np.argsort(ends)[-6:].tolist()}")
if os.environ.get("TRACE_DUMP"):
    np.save(os.environ["TRACE_DUMP"], tr)
n = int((tr[4] > 0).sum())


def st(name, v):
    v = v[np.isfinite(v)]
    if v.size == 0:
        return
    print(f"  {name:40s} mean {np.mean(v):9.1f}  p50 {np.median(v):9.1f}  p90 {np.percentile(v, 90):9.1f}")


def diff(a, b):
    m = (tr[a] != 0) & (tr[b] != 0)
    return (tr[b] - tr[a])[m][2:-2].astype(float)


base = tr[8][0]


def d(a, b, i):
    return int(tr[b][i] - tr[a][i]) if tr[a][i] and tr[b][i] else None
print("  tile | start +data +buf +bar +done | mma: +afull_seen(after done) +issued | release(pair) after issue")
for i in range(100, 116):
    rel = int(tr[15][i // 2] - tr[7][i | 1]) if tr[15][i // 2] and tr[7][i | 1] else None
    print("  %4d | %7d %+5s %+5s %+5s %+5s | %+6s %+5s | %+6s" % (i, tr[13][i] - base, d(13, 14, i), d(14, 0, i), d(0, 1, i),
          d(1, 2, i), d(2, 4, i), d(4, 7, i), rel))
st("mma: iteration (s8[i+1]-s8[i])", np.diff(tr[8][:n].astype(float))[2:-2])
st("decode: start->data", diff(13, 14))
st("decode: data->buffer", diff(14, 0))
st("decode: buffer->barrier", diff(0, 1))
st("decode: barrier->done", diff(1, 2))
if os.environ.get("TRACE_RAW"):
    print("  tile |  top(8)  xfull  afull  issue  next | decoded(2) before afull_seen")
    idx = [i for i in range(100, 160) if tr[8][i]]
    for i, j in zip(idx[:-1], idx[1:]):
        print("  %4d | %7d %6d %6d %6d %5d | %7d" % (i, tr[8][i] - base, tr[3][i] - tr[8][i], tr[4][i] - tr[3][i],
              tr[7][i] - tr[4][i] if tr[7][i] else -1, tr[8][j] - tr[7][i] if tr[7][i] else -1,
              tr[4][i] - tr[2][i] if tr[2][i] else 0))
if os.environ.get("TRACE_CHAIN"):
    na = int(os.environ.get("TRACE_NA", "8"))
    print("  tile | decoded  +mma_sees  +issued  +released  +woken(t+NA) | decode_start->done")
    for i in range(100, 130):
        print("  %4d | %7d %9d %8d %10d %12d | %7d" % (
            i, tr[2][i] - base, tr[4][i] - tr[2][i], tr[7][i] - tr[4][i], tr[15][i] - tr[7][i],
            tr[0][i + na] - tr[15][i] if tr[0][i + na] else -1, tr[2][i] - tr[13][i]))
if os.environ.get("TRACE_START"):
    k0 = tr[9][0]
    print("  kernel start -> unit table ready %d, first chunk issued %d, first meta published %d, first decode start %d,"
          " first MMA %d, last MMA commit %d (cycles)" % (tr[9][1] - k0, tr[6][0] - k0, tr[10][0] - k0, tr[13][0] - k0,
                                                          tr[8][0] - k0, tr[7][n - 1] - k0 if n else -1))
