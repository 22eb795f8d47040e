"""Debug tool: fixed per-launch cost of K2. Times tiny SpMMs (one or a few tiles per
CTA) back to back in a CUDA graph (hot) and after a 256 MB read (cold), so the
intercept of the per-tile model can be split from the per-tile cost.
  python tools/fixed_cost.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_10285_b200 as tc  # noqa: E402

flush = torch.zeros(32 * 1024 * 1024, dtype=torch.int64, device="cuda")
sink = torch.empty((), dtype=torch.int64, device="cuda")
R = 16


def graph_time(fn, with_flush):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(R):
            if with_flush:
                torch.sum(flush, dim=0, out=sink)
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / R


t_flush = graph_time(lambda: None, True)
for (m, k, n, beta, split) in [(256, 64, 16, 0.9, 1), (256, 640, 16, 0.9, 1), (256, 6400, 16, 0.9, 1),
                               (18944, 64, 16, 0.9, 1), (18944, 640, 16, 0.9, 1), (18944, 6400, 16, 0.9, 1),
                               (18944, 6400, 16, 0.7, 1), (9216, 9216, 8, 0.9, 2), (9216, 9216, 8, 0.9, 1)]:
    w = tc.gen_synthetic(m, k, beta, 1)
    x = tc.gen_synthetic(k, n, 0.0, 2)
    t = tc.encode(w)
    y = torch.empty((m, n), device="cuda")
    ws = tc.SpmmWorkspace()
    f = lambda: tc.spmm(t, x, split_k=split, out=y, ws=ws, check=False)  # noqa: E731
    hot = graph_time(f, False)
    cold = graph_time(f, True) - t_flush
    tiles_cta = -(-((m + 127) // 128 + 1) // 2 // 74) * ((k + 63) // 64) if split == 1 else None
    print(f"m={m:6d} k={k:5d} n={n} beta={beta} split={split}: hot {hot:7.2f} us  cold {cold:7.2f} us")
