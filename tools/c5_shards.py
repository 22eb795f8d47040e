"""Per-rank compute of BASELINE configs[4] on one GPU: the row shard a rank of a G-GPU
row-sharded run holds (OPT-175B FFN1 49152x12288, 80 %, N=32), timed like bench.py's
cells (cold L2, R replays per event pair), for G = 1, 2, 4, 8. Prints the kernel-only
scaling T(1) / T(shard of G) — the ceiling of the multi-GPU speed-up before the
exchange of Y.   python tools/c5_shards.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_10285_b200 as tc  # noqa: E402
from paper_2309_10285_b200.sharding import shard_plan  # noqa: E402

M, K, N, beta = 49152, 12288, 32, 0.8
w = tc.gen_synthetic(M, K, beta, 1)
x = tc.gen_synthetic(K, N, 0.0, 2)
t = tc.encode(w)
del w
flush = torch.zeros(32 * 1024 * 1024, dtype=torch.int64, device="cuda")
sink = torch.empty((), dtype=torch.int64, device="cuda")
R = 8


def timed(fn):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(R):
            torch.sum(flush, dim=0, out=sink)
            fn()
    out = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3 / R)
    return float(np.median(out))


gf = torch.cuda.CUDAGraph()
with torch.cuda.graph(gf):
    for _ in range(R):
        torch.sum(flush, dim=0, out=sink)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
gf.replay()
b.record()
torch.cuda.synchronize()
t_flush = a.elapsed_time(b) * 1e3 / R
res = {}
for G in (1, 2, 4, 8):
    sh = shard_plan(M, 128, G)[0]
    local = tc.shard_rows(t, sh.tr0, sh.tr1)
    y = torch.empty((sh.rows, N), dtype=torch.float32, device="cuda")
    ws = tc.SpmmWorkspace()
    us = timed(lambda: tc.spmm(local, x, out=y, ws=ws, check=False)) - t_flush
    res[G] = {"rows": sh.rows, "split": tc.auto_split(sh.rows, K, N), "us": round(us, 2)}
for G in res:
    res[G]["kernel_only_scaling"] = round(res[1]["us"] / res[G]["us"], 2)
print(json.dumps({"config": "OPT-175B FFN1 49152x12288 beta=0.8 N=32 (configs[4]); rank 0's shard per G",
                  "shards": res}))
