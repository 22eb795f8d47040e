"""Benchmark of the B200 Tiled-CSL SpMM (Flash-LLM LSCD) against BASELINE.json.

Workload (BASELINE.json metric "SpMM TFLOPS (2MKN/t) + HBM GB/s, OPT-66B/175B
shapes, N=8-64, 70-90% sparse"): configs[1] — the four OPT-66B decoder MatMuls
(QKV 27648x9216, out 9216x9216, FFN1 36864x9216, FFN2 9216x36864) — and
configs[3] — the three OPT-175B MatMuls (QKV 36864x12288, FFN1 49152x12288, FFN2
12288x49152) — at N = 8/16/32/64 and 70/80/90 % sparsity: 84 SpMMs per step.

Inputs are the reference's own generator bits: W = gen_random_sparse(M, K, beta,
seed 1), X = gen_random_sparse(K, N, 0, seed 2) (proj/src/matrix.cpp:35-67), made
by the drop-in host library (libtcsl.so, bit-identical to the reference; the GPU
parity tests check these exact inputs against the CPU oracle), encoded on the GPU.
Metric: TFLOPS = sum 2MKN / time (dense-equivalent), plus GB/s of
the algorithmic bytes 4E + 4(T+1) + 2KN + 4MN.

  python bench.py [--gpus N --steps K --warmup W]          # our arm
  python bench.py --impl reference [...]                    # reference CPU arm
Under torchrun (N > 1) every matrix is row-sharded across the ranks and Y is
all-gathered through the C-ABI's NCCL entry point (BASELINE.json north_star (4));
rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMM TFLOPS (2MKN/t) + HBM GB/s, OPT-66B/175B shapes, N=8-64, 70-90% sparse"
SHAPES_66B = {"qkv": (27648, 9216), "out": (9216, 9216), "ffn1": (36864, 9216), "ffn2": (9216, 36864)}
SHAPES_175B = {"qkv175": (36864, 12288), "ffn1_175": (49152, 12288), "ffn2_175": (12288, 49152)}
SUITES = {
    "all": ({**SHAPES_66B, **SHAPES_175B},
            "OPT-66B (configs[1]) + OPT-175B (configs[3]) SpMMs: 7 shapes x N{8,16,32,64} x sparsity{0.7,0.8,0.9} "
            "(84 per step)"),
    "opt66b": (SHAPES_66B, "OPT-66B QKV/out/FFN1/FFN2 SpMMs x N{8,16,32,64} x sparsity{0.7,0.8,0.9} (48 per step)"),
    "opt175b": (SHAPES_175B, "OPT-175B QKV/FFN1/FFN2 SpMMs x N{8,16,32,64} x sparsity{0.7,0.8,0.9} (36 per step)"),
    "c1": ({"c1": (7168, 7168)}, "OPT-30B attn-out 7168x7168 (configs[0]; use --only c1:0.8:16)"),
}
SHAPES, WORKLOAD = SUITES["all"]
NS = [8, 16, 32, 64]
BETAS = [0.7, 0.8, 0.9]
SEED_W, SEED_X = 1, 2
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM, FALLBACK_TC = 6650.0, 1590.0  # B200_PROFILING.md fallbacks (GB/s, dense bf16 TF/s)
CPU_ROWS_PER_THREAD = 128


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, FALLBACK_TC, "fallback (B200_PROFILING.md)"


def parse_only(spec):
    """--only qkv:0.8:16,ffn2:0.9:8 -> [(name, beta, n)]"""
    cells = []
    for part in spec.split(","):
        name, beta, n = part.split(":")
        cells.append((name, float(beta), int(n)))
    return cells


def cell_list(args):
    """N outermost: between two uses of one compressed weight every other weight of
    the step streams through HBM, so no cell reads its weight from L2."""
    if args.only:
        return parse_only(args.only)
    return [(name, beta, n) for n in NS for beta in BETAS for name in SHAPES]


def weight_list(cells):
    seen = []
    for name, beta, _ in cells:
        if (name, beta) not in seen:
            seen.append((name, beta))
    return seen


def alg_bytes(t, n):
    return 4 * t.n_entries + 4 * (t.num_tiles + 1) + 2 * t.k * n + 4 * t.m * n


def flops_of(m, k, n):
    return 2.0 * m * k * n


def bench_config(args, world):
    """The `config` object of the JSON line; identical for both arms (the reference
    arm's sampling is described in its cpu_baseline.sample)."""
    return {"workload": WORKLOAD, "tile": "128x64 Tiled-CSL, bank-reordered", "n_cells": len(cell_list(args)),
            "inputs": "gen_random_sparse(M,K,beta,seed 1), X = gen_random_sparse(K,N,0,seed 2)",
            "l2": "cold: cells run N-outer, so each compressed weight is re-read only after every other weight "
                  "of the step (GBs) has streamed; per-cell times read a 256 MB buffer (2x L2) before each replay",
            "parallelism": "single GPU" if world == 1 else f"row-shard x{world} + NCCL all-gather of Y (C-ABI)"}


# ------------------------------------------------------------------------------ host inputs
_host_lib = None


def host_lib():
    """The C++ drop-in host library (its C entry point, include/tcsl_host.h)."""
    global _host_lib
    if _host_lib is None:
        path = os.path.join(ROOT, "paper_2309_10285_b200", "_lib", "libtcsl.so")
        L = C.CDLL(path)
        L.tcsl_host_gen_random_sparse.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_void_p]
        L.tcsl_host_gen_random_sparse.restype = C.c_int
        _host_lib = L
    return _host_lib


def gen_random_sparse(rows, cols, beta, seed):
    out = np.empty((rows, cols), np.uint16)
    st = host_lib().tcsl_host_gen_random_sparse(rows, cols, beta, seed, out.ctypes.data)
    if st:
        raise RuntimeError(f"gen_random_sparse failed ({st})")
    return out


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML SM-clock / throttle-reason sampler running during the timed region."""

    NAMES = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
             0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index=0, period=0.005):
        self.samples, self.reasons, self.period = [], set(), period
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.NAMES.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def ncu_traffic():
    """DRAM bytes per launch of the SpMM kernel from the newest committed ncu --set full
    summary of the reference cell (profiles/*_ncu_*ffn1_b08_n16.json), or None."""
    import glob
    import re

    def version(path):  # r02_ncu_v3_ffn1_b08_n16.json -> (2, 3)
        m = re.search(r"r(\d+)_ncu_v(\d+)[a-z]?_", os.path.basename(path))
        return (int(m.group(1)), int(m.group(2))) if m else (-1, -1)

    files = [f for f in glob.glob(os.path.join(ROOT, "profiles", "*_ncu_*.json")) if "_ffn1_b08_n16" in f]
    if not files:
        return None
    try:
        path = sorted(files, key=version)[-1]
        with open(path) as f:
            d = json.load(f)
        return {"dram_bytes_per_launch": d["dram_bytes_per_launch"], "alg_bytes_per_launch": d["alg_bytes_per_launch"],
                "cell": d.get("cell", ""), "source": os.path.relpath(path, ROOT)}
    except Exception:
        return None


# ------------------------------------------------------------------------------ our arm
def prepare_weights(tc, torch, dev, weights, rank, world, keep_rows):
    """Generate every weight on the host (reference generator, a thread per weight),
    upload, encode on the GPU (K1) and keep its row shard. Returns the shards, the K1
    timings and the first `keep_rows` rows of each weight (for the CPU baseline)."""
    from paper_2309_10285_b200.sharding import shard_plan

    def gen(key):
        m, k = SHAPES[key[0]]
        return gen_random_sparse(m, k, key[1], SEED_W)

    mats, enc, head = {}, {}, {}
    workers = max(1, min(len(weights), cpu_threads() // max(1, world)))
    with ThreadPoolExecutor(max_workers=workers) as ex:
        futs = {key: ex.submit(gen, key) for key in weights}
        for key in weights:
            a = futs.pop(key).result()
            m, k = SHAPES[key[0]]
            plan = shard_plan(m, 128, world)
            sh = plan[rank]
            if keep_rows:
                head[key] = a[:keep_rows].copy()
            w = torch.from_numpy(a[sh.row0:sh.row0 + sh.rows].view(np.int16)).to(dev)
            del a
            tc.encode(w)  # warm (allocations, tensor-map setup)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t = tc.encode(w)
            e1.record()
            torch.cuda.synchronize()
            enc_us = e0.elapsed_time(e1) * 1e3
            # one-pass encoder (W read once) into a buffer of known capacity; same bits
            tc.encode(w, capacity=t.n_entries)
            torch.cuda.synchronize()
            e0.record()
            tf = tc.encode(w, capacity=t.n_entries)
            e1.record()
            torch.cuda.synchronize()
            us_f = e0.elapsed_time(e1) * 1e3
            if not (torch.equal(tf.offsets, t.offsets) and torch.equal(tf.entries, t.entries)):
                raise RuntimeError(f"fused encoder differs from count+emit on {key}")
            del tf
            enc[key] = (enc_us, 2 * w.numel(), t.n_entries, us_f)
            mats[key] = (t, sh, plan)
            del w
    return mats, enc, head


def run_ours(args, rank, world):
    import torch

    import paper_2309_10285_b200 as tc
    from paper_2309_10285_b200.sharding import allgather_rows

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cells = cell_list(args)
    weights = weight_list(cells)
    hbm_peak, tc_peak, peak_kind = peaks()
    threads = max(1, min(cpu_threads(), 64))
    keep_rows = threads * CPU_ROWS_PER_THREAD if (rank == 0 and world == 1 and not args.no_cpu_baseline) else 0
    mats, enc, head = prepare_weights(tc, torch, dev, weights, rank, world, keep_rows)

    comm = tc.RowComm(rank, world) if world > 1 else None
    xs, ys, gathered, wss, hx = {}, {}, {}, {}, {}
    for name, beta, n in cells:
        M, K = SHAPES[name]
        if (K, n) not in xs:
            hx[(K, n)] = gen_random_sparse(K, n, 0.0, SEED_X)
            xs[(K, n)] = torch.from_numpy(hx[(K, n)].view(np.int16)).to(dev)
        t, sh, plan = mats[(name, beta)]
        ys[(name, beta, n)] = torch.empty((t.m, n), dtype=torch.float32, device=dev)
        wss[(name, beta, n)] = tc.SpmmWorkspace()
        if world > 1:
            gathered[(name, beta, n)] = torch.empty((world * max(s.rows for s in plan), n), dtype=torch.float32,
                                                    device=dev)

    def one_cell(name, beta, n):
        t, sh, plan = mats[(name, beta)]
        y = ys[(name, beta, n)]
        tc.spmm(t, xs[(SHAPES[name][1], n)], split_k=args.split, out=y, ws=wss[(name, beta, n)], check=False)
        if world > 1:
            allgather_rows(y, plan, comm=comm, out=gathered[(name, beta, n)])

    def step():
        for c in cells:
            one_cell(*c)

    # correctness gate before timing: device error words clean
    for c in cells:
        t = mats[(c[0], c[1])][0]
        tc.spmm(t, xs[(SHAPES[c[0]][1], c[2])], split_k=args.split, out=ys[c], ws=wss[c], check=True)
    torch.cuda.synchronize()

    graph = None
    if not args.no_graph:
        step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()
    run = graph.replay if graph is not None else step

    for _ in range(max(3, args.warmup)):
        run()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clocks:
        torch.cuda.synchronize()
        start.record()
        for _ in range(args.steps):
            run()
        end.record()
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = start.elapsed_time(end) / args.steps
    if world > 1:
        tms = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(tms, op=torch.distributed.ReduceOp.MAX)
        ms = float(tms.item())

    flops = sum(flops_of(*SHAPES[nm], n) for nm, b, n in cells)
    launches_per_step = 0
    for nm, b, n in cells:
        t = mats[(nm, b)][0]
        launches_per_step += 1 + ((args.split or tc.auto_split(t.m, t.k, n)) > 1)
    total_alg = sum(alg_bytes(mats[(nm, b)][0], n) for nm, b, n in cells)

    result = {
        "metric": METRIC,
        "value": round(flops / (ms * 1e-3) / 1e12, 3),
        "unit": "TFLOPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f16 in / f32 accumulate / f32 out",
        "data": "synthetic: the reference's gen_random_sparse bits (seeds 1 / 2) via the drop-in host library",
        "config": bench_config(args, world),
        "hbm_gbs": round(total_alg / (ms * 1e-3) / 1e9, 1),
        "gpu_launches": launches_per_step * args.steps + (len(cells) * args.steps if world > 1 else 0),
        "clocks": clocks.summary(),
    }
    if world > 1 or args.quick:
        return result

    # ---- per-SpMM device times, cold: each replay is preceded by a 256 MB read (2x L2, clean
    # lines, so no write-back lands in the cell). t_cell = (T[read+cell] - T[read]) / R over
    # R replays inside one event pair (well above the ~2 us timer quantum).
    flush = torch.zeros(32 * 1024 * 1024, dtype=torch.int64, device=dev)  # 256 MB, read-only below
    sink = torch.empty((), dtype=torch.int64, device=dev)
    R = max(4, args.kernel_reps)

    def read_flush():
        torch.sum(flush, dim=0, out=sink)

    def graph_of(fn, reps):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                fn()
        return g

    def timed(g, reps=3):
        out = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(out)

    g_flush = graph_of(read_flush, R)
    t_flush = timed(g_flush, 5) / R
    cell_rows, sum_t, sum_bytes = [], 0.0, 0
    for nm, b, n in cells:
        t = mats[(nm, b)][0]
        g = graph_of(lambda: (read_flush(), one_cell(nm, b, n)), R)
        us = max(timed(g) / R - t_flush, 1e-3)
        del g
        nbytes = alg_bytes(t, n)
        fl = flops_of(t.m, t.k, n)
        t_hbm = nbytes / (hbm_peak * 1e3)  # us
        t_tc = fl / (tc_peak * 1e6)
        cell_rows.append({"shape": nm, "M": t.m, "K": t.k, "N": n, "sparsity": b, "E": t.n_entries,
                          "split": args.split or tc.auto_split(t.m, t.k, n), "us": round(us, 2),
                          "tflops": round(fl / us / 1e6, 2), "gbs": round(nbytes / us / 1e3, 1),
                          "hbm_frac": round(t_hbm / us, 3), "roofline_frac": round(max(t_hbm, t_tc) / us, 3)})
        est = tc.estimate(t.m, t.k, n, t.n_entries, cell_rows[-1]["split"], hbm_peak)
        cell_rows[-1]["model_us"] = round(est["us"], 2)
        cell_rows[-1]["model_bound"] = est["bound"]
        sum_t += us
        sum_bytes += nbytes
    torch.cuda.synchronize()

    # ---- cuBLAS dense fp16 on the same shapes (context only; the same cold protocol)
    if not args.no_cublas:
        for nm in SHAPES:
            if not any(r["shape"] == nm for r in cell_rows):
                continue
            M, K = SHAPES[nm]
            wd = torch.randn((M, K), dtype=torch.float16, device=dev)
            for row in cell_rows:
                if row["shape"] != nm:
                    continue
                x = xs[(K, row["N"])].view(torch.float16)
                yd = torch.empty((M, row["N"]), dtype=torch.float16, device=dev)
                torch.matmul(wd, x, out=yd)  # cuBLAS handle / workspace before capture
                torch.cuda.synchronize()
                g = graph_of(lambda: (read_flush(), torch.matmul(wd, x, out=yd)), R)
                row["cublas_dense_fp16_us"] = round(max(timed(g) / R - t_flush, 1e-3), 2)
                row["speedup_vs_cublas"] = round(row["cublas_dense_fp16_us"] / row["us"], 2)
                del g
            del wd
    del flush

    traffic = ncu_traffic()
    achieved = sum_bytes / sum_t / 1e3
    by_beta = {}
    for b in BETAS:
        rows = [r for r in cell_rows if r["sparsity"] == b]
        if rows and sum(r["us"] for r in rows) > 0:  # (per-cell times are ~0 under a serialising profiler)
            by_beta[str(b)] = round(sum(r["gbs"] * r["us"] for r in rows) / sum(r["us"] for r in rows) / hbm_peak, 3)
    result["roofline"] = {
        "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
        "frac": round(achieved / hbm_peak, 3), "traffic": (traffic or {}).get("dram_bytes_per_launch"),
        "traffic_detail": traffic, "peak_kind": peak_kind,
        "kernel": "tcsl spmm_sm100_kernel (+ split-K reduce when split>1)",
        "bytes_per_launch": "4E + 4(T+1) + 2KN + 4MN (SURVEY.md §8d), per cell; achieved = sum bytes / sum cold us",
        "frac_by_sparsity": by_beta,
        "max_hbm_tc_frac": round(sum(r["roofline_frac"] * r["us"] for r in cell_rows) / sum_t, 3),
        "sum_cold_cell_ms": round(sum_t / 1e3, 4),
    }
    result["cells"] = cell_rows
    rel = sorted(abs(r["model_us"] - r["us"]) / r["us"] for r in cell_rows)
    result["model"] = {
        "what": "a-priori B200 time model tcsl_cuda_spmm_estimate (fixed + max(HBM, tensor, smem, chain)) vs the "
                "cold per-cell times",
        "median_rel_err": round(rel[len(rel) // 2], 4), "max_rel_err": round(rel[-1], 4),
        "bounds": {b: sum(r["model_bound"] == b for r in cell_rows) for b in ("hbm", "tensor", "smem", "chain")},
    }
    result["encoder"] = {
        "kernel": "K1 tcsl_cuda_encode_count + scan + encode_emit (bit-exact Tiled-CSL)",
        "weights": len(enc), "ms_total": round(sum(v[0] for v in enc.values()) / 1e3, 3),
        "dense_gbs": round(sum(v[1] for v in enc.values()) / (sum(v[0] for v in enc.values()) * 1e3), 1),
        "per_weight_us": {f"{k[0]}@{k[1]}": round(v[0], 1) for k, v in enc.items()},
        "fused": {
            "kernel": "K1 tcsl_cuda_encode_fused: one pass (W read once), decoupled look-back offsets",
            "ms_total": round(sum(v[3] for v in enc.values()) / 1e3, 3),
            "dense_gbs": round(sum(v[1] for v in enc.values()) / (sum(v[3] for v in enc.values()) * 1e3), 1),
            "hbm_gbs": round(sum(v[1] + 4 * v[2] for v in enc.values()) / (sum(v[3] for v in enc.values()) * 1e3), 1),
            "per_weight_us": {f"{k[0]}@{k[1]}": round(v[3], 1) for k, v in enc.items()},
            "bit_identical_to_two_pass": True,
        },
    }
    if not args.no_e2e:
        result["e2e"] = run_e2e(args, tc, torch, mats, hx, cells, dev)
    if not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(head, cells, threads, steps=1)
    return result


def run_e2e(args, tc, torch, mats, hx, cells, dev):
    """Through the public API with HOST buffers: every step uploads each cell's X from
    pinned host memory, runs spmm on the resident weights and reads Y back into pinned
    host memory (the serving call: weights are model state loaded once, e.g. with
    paper_2309_10285_b200.load_tcsl). Uploads, SpMMs and read-backs run on three
    streams ordered by events, so PCIe traffic of one cell overlaps the kernel of
    another. The drop-in variant that also re-uploads the compressed weights on
    every call (tcsl::spmm's host TcslMatrix) is reported beside it."""
    hxp = {k: torch.from_numpy(v.view(np.int16)).pin_memory() for k, v in hx.items()}
    xdev = {c: torch.empty(hxp[(SHAPES[c[0]][1], c[2])].shape, dtype=torch.int16, device=dev) for c in cells}
    ydev = {c: torch.empty((mats[(c[0], c[1])][0].m, c[2]), dtype=torch.float32, device=dev) for c in cells}
    hy = {c: torch.empty((mats[(c[0], c[1])][0].m, c[2]), dtype=torch.float32).pin_memory() for c in cells}
    ws = tc.SpmmWorkspace()
    flops = sum(flops_of(*SHAPES[nm], n) for nm, b, n in cells)
    h2d = sum(2 * hxp[(SHAPES[nm][1], n)].numel() for nm, b, n in cells)
    d2h = sum(4 * hy[c].numel() for c in cells)
    compute = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()

    def step_resident():
        ev_x, ev_y = {}, {}
        with torch.cuda.stream(up):
            for c in cells:
                xdev[c].copy_(hxp[(SHAPES[c[0]][1], c[2])], non_blocking=True)
                ev_x[c] = torch.cuda.Event()
                ev_x[c].record(up)
        for c in cells:
            compute.wait_event(ev_x[c])
            t = mats[(c[0], c[1])][0]
            tc.spmm(t, xdev[c], ws=ws, out=ydev[c], check=False)
            ev_y[c] = torch.cuda.Event()
            ev_y[c].record(compute)
        with torch.cuda.stream(down):
            for c in cells:
                down.wait_event(ev_y[c])
                hy[c].copy_(ydev[c], non_blocking=True)
        down.synchronize()
        compute.synchronize()

    for _ in range(2):
        step_resident()
    steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(steps):
        step_resident()
    ms = (time.perf_counter() - t0) / steps * 1e3
    out = {"value": round(flops / (ms * 1e-3) / 1e12, 3), "unit": "TFLOPS", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 3), "steps": steps, "clock": "host wall clock",
           "api": "paper_2309_10285_b200.spmm (tcsl_cuda_spmm_ex): X pinned host -> device, Y device -> pinned "
                  "host every call; weights resident; copies on two side streams overlap the kernels"}

    # drop-in tcsl::spmm semantics: the compressed weights cross PCIe on every call too
    host = {key: (v[0].offsets.cpu().pin_memory(), v[0].entries.cpu().pin_memory()) for key, v in mats.items()}
    maxE = max(v[0].n_entries for v in mats.values())
    maxT = max(v[0].num_tiles for v in mats.values())
    d_ent = torch.empty(maxE, dtype=torch.int32, device=dev)
    d_off = torch.empty(maxT + 1, dtype=torch.int32, device=dev)
    h2d_full = h2d + sum(4 * (host[(nm, b)][0].numel() + host[(nm, b)][1].numel()) for nm, b, n in cells)

    def step_upload():
        for nm, b, n in cells:
            t = mats[(nm, b)][0]
            off, ent = host[(nm, b)]
            d_off[:off.numel()].copy_(off, non_blocking=True)
            d_ent[:ent.numel()].copy_(ent, non_blocking=True)
            xd = xdev[(nm, b, n)]
            xd.copy_(hxp[(t.k, n)], non_blocking=True)
            # a fresh host-provided matrix: spmm validates it on the device (one pass over E)
            tt = tc.TcslMatrix(t.m, t.k, t.cfg, t.reordered, d_off[:off.numel()], d_ent[:ent.numel()])
            y = tc.spmm(tt, xd, ws=ws, check=False)
            hy[(nm, b, n)].copy_(y, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    step_upload()
    t0 = time.perf_counter()
    step_upload()
    ms_u = (time.perf_counter() - t0) * 1e3
    out["weights_uploaded_per_call"] = {"value": round(flops / (ms_u * 1e-3) / 1e12, 4), "unit": "TFLOPS",
                                        "h2d_bytes_per_step": h2d_full, "d2h_bytes_per_step": d2h,
                                        "ms_per_step": round(ms_u, 3), "steps": 1}
    return out


# ------------------------------------------------------------------------------ CPU side
def cpu_sample_desc(nrows, threads, ncells):
    return (f"{ncells} cells (every cell of the step), the first {nrows} rows of each weight "
            f"(one 128-row block per thread), unmodified reference tcsl::spmm per row block; host: {cpu_model()}, "
            f"{cpu_threads()} hardware threads, {threads} used")


def cpu_baseline(head, cells, threads, steps=1):
    """The reference's CPU tcsl::spmm (oracle/_ref: the unmodified reference sources;
    else the C port) on a bounded sample of this workload: the first threads*128 rows
    of every weight, every cell, one 128-row block per thread."""
    import oracle
    kind = "reference" if oracle.ref_available() else "port"
    impl = oracle.ref() if kind == "reference" else oracle.port()
    plans, xs = {}, {}
    for key, a in head.items():
        t = impl.encode(a)
        plans[key] = (impl.spmm_plan(t, threads), a.shape[0]) if kind == "reference" else (t, a.shape[0])
    for name, beta, n in cells:
        K = SHAPES[name][1]
        if (K, n) not in xs:
            xs[(K, n)] = gen_random_sparse(K, n, 0.0, SEED_X)
    total_fl, total_s = 0.0, 0.0
    for _ in range(steps):
        for name, beta, n in cells:
            plan, rows = plans[(name, beta)]
            x = xs[(SHAPES[name][1], n)]
            y = np.empty((rows, n), np.float32)
            t0 = time.perf_counter()
            if kind == "reference":
                impl.spmm_run(plan, x, rows, y)
            else:
                impl.spmm(plan, x, threads)
            total_s += time.perf_counter() - t0
            total_fl += flops_of(rows, SHAPES[name][1], n)
    if kind == "reference":
        for plan, _ in plans.values():
            impl.spmm_free(plan)
    nrows = next(iter(head.values())).shape[0]
    return {"value": round(total_fl / total_s / 1e12, 6), "unit": "TFLOPS", "cores": threads, "kind": kind,
            "sample": cpu_sample_desc(nrows, threads, len(cells)), "seconds": round(total_s, 2), "steps": steps}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref), on this arm's workload sample, all host threads."""
    if rank != 0:
        return None
    cells = cell_list(args)
    weights = weight_list(cells)
    threads = max(1, min(cpu_threads(), 64))
    nrows = threads * CPU_ROWS_PER_THREAD

    def gen(key):
        m, k = SHAPES[key[0]]
        return key, gen_random_sparse(m, k, key[1], SEED_W)[:nrows].copy()

    with ThreadPoolExecutor(max_workers=threads) as ex:
        head = dict(ex.map(gen, weights))
    steps = max(1, min(args.steps, 3))
    t_start = time.perf_counter()
    base = cpu_baseline(head, cells, threads, steps=steps)
    ms = (time.perf_counter() - t_start) / steps * 1e3
    value = base["value"]
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world,
            "steps": steps, "warmup": 0, "ms_per_step": round(ms, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (fp16 inputs widened exactly, f32 accumulate)",
            "data": "synthetic: the reference's gen_random_sparse bits (seeds 1 / 2)",
            "config": bench_config(args, 1),
            "cpu_baseline": base,
            "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    global SHAPES, WORKLOAD
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--suite", default="all", choices=sorted(SUITES),
                    help="all = configs[1] + configs[3] (the metric's shapes); opt66b / opt175b = one of them")
    ap.add_argument("--only", default="", help="cells as shape:beta:n,... (e.g. ffn2:0.9:8)")
    ap.add_argument("--split", type=int, default=0, help="force split-K S (0 = auto; SURVEY §8d C3)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="headline only (no per-cell, e2e, cuBLAS, CPU legs)")
    ap.add_argument("--kernel-reps", type=int, default=8)
    args = ap.parse_args()
    SHAPES, WORKLOAD = SUITES[args.suite]
    if args.only:
        SHAPES = {**SHAPES_66B, **SHAPES_175B, **SUITES["c1"][0]}

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    res = run_ours(args, rank, world)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
