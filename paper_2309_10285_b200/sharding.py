"""Row (M) sharding of one Tiled-CSL weight across the GPUs of a node
(BASELINE.json north_star (4)).

A shard is the contiguous range of tile rows [tr0, tr1): because tiles are
stored row-major over the tile grid (proj/src/tcsl_format.cpp:56-57), its
tiles are the contiguous range [tr0*tk, tr1*tk) and its entries the contiguous
range [off[tr0*tk], off[tr1*tk]); rebasing the offsets gives exactly the
Tiled-CSL that `encode` would produce for those rows (checked in the tests).
X is replicated; each rank computes its rows of Y, and one all-gather (NCCL
over NVLink on GPUs, gloo on CPU) assembles Y in rank order. No other
collective exists on this path.

Fused alternative (push=True): Y lives in symmetric memory (one full-Y buffer
per rank, peer-mapped over NVLink); the SpMM epilogue stores every finished
row block straight into all ranks' buffers (tcsl_cuda_spmm_push), so the
exchange overlaps the SpMM tile by tile and only a device-side barrier
(symmetric-memory signal pads) follows the kernel.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    tr0: int      # first tile row
    tr1: int      # one past the last tile row
    row0: int     # first matrix row
    rows: int     # rows in this shard (the last one may be ragged)


def shard_plan(m: int, m_tb: int, world: int) -> list[Shard]:
    """Balanced contiguous tile-row ranges, one per rank (empty ranges allowed)."""
    tiles_m = -(-m // m_tb)
    out = []
    for r in range(world):
        tr0, tr1 = tiles_m * r // world, tiles_m * (r + 1) // world
        row0 = tr0 * m_tb
        rows = max(0, min(m, tr1 * m_tb) - row0)
        out.append(Shard(r, tr0, tr1, row0, rows))
    return out


def slice_rows(offsets: np.ndarray, entries: np.ndarray, tiles_k: int, shard: Shard):
    """Host slice of a Tiled-CSL matrix: (rebased offsets, entry view)."""
    t0, t1 = shard.tr0 * tiles_k, shard.tr1 * tiles_k
    off = np.asarray(offsets, dtype=np.uint32)[t0:t1 + 1]
    lo, hi = int(off[0]), int(off[-1])
    return (off - off[0]).astype(np.uint32), np.asarray(entries, dtype=np.uint32)[lo:hi]


def max_rows(plan: list[Shard]) -> int:
    return max(s.rows for s in plan)


def allgather_rows(y_local, plan: list[Shard], group=None, comm=None, out=None):
    """All-gather row shards of Y (torch tensors, [rows_r, n]) into the full Y.

    comm: a paper_2309_10285_b200.RowComm — the C-ABI's tcsl_cuda_allgather_rows
    (one ncclAllGather, stream-ordered). Without it, torch.distributed on `group`
    (NCCL or gloo). When every shard has the same row count (m / G a multiple of
    128, as in BASELINE configs[4]) the gathered buffer IS Y (rank-major rows) and
    no copy is made; ragged plans pad to the largest shard and drop the padding."""
    import torch
    import torch.distributed as dist

    world = len(plan)
    n = y_local.shape[1]
    rmax = max_rows(plan)
    uniform = all(s.rows == rmax for s in plan)
    if uniform:
        pad = y_local
        full = out if out is not None else torch.empty((world * rmax, n), dtype=y_local.dtype, device=y_local.device)
    else:
        pad = torch.zeros((rmax, n), dtype=y_local.dtype, device=y_local.device)
        pad[: y_local.shape[0]].copy_(y_local)
        full = torch.empty((world * rmax, n), dtype=y_local.dtype, device=y_local.device)
    if comm is not None:
        comm.allgather_rows(pad, full)
    elif dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, pad, group=group)
    else:
        dist.all_gather(list(full.chunk(world)), pad, group=group)
    if uniform:
        return full
    parts = [full[s.rank * rmax: s.rank * rmax + s.rows] for s in plan]
    return torch.cat(parts, dim=0)


def push_targets(buffer_ptrs, plan: list[Shard], rank: int, n: int, elem_bytes: int) -> list[int]:
    """Device addresses the fused epilogue writes rank `rank`'s rows to: its row
    block (rank * rmax rows in) inside every rank's full-Y buffer (rank-major,
    rmax rows per rank, row stride n)."""
    rmax = max_rows(plan)
    return [int(p) + rank * rmax * n * elem_bytes for p in buffer_ptrs]


class RowShardedSpmm:
    """One rank's part of a row-sharded SpMM on the GPU: holds the rank's
    Tiled-CSL shard (device), runs the tcgen05 SpMM on it and all-gathers Y —
    after the kernel (NCCL / torch.distributed), or fused into its epilogue
    (push=True: symmetric-memory Y, tcsl_cuda_spmm_push, device barrier)."""

    def __init__(self, t_full, world: int, rank: int, group=None, comm=None, push: bool = False):
        from . import shard_rows
        self.plan = shard_plan(t_full.m, t_full.cfg.m_tb, world)
        self.shard = self.plan[rank]
        self.rank = rank
        self.group = group
        self.comm = comm  # RowComm: the C-ABI NCCL all-gather (else torch.distributed)
        self.push = push
        self._symm = {}  # (n, dtype) -> (full-Y symmetric buffer, handle, device peer table)
        self.local = shard_rows(t_full, self.shard.tr0, self.shard.tr1) if self.shard.rows else None
        self.m = t_full.m

    def _push_buffer(self, n, dtype, device):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        key = (n, dtype)
        if key not in self._symm:
            rmax = max_rows(self.plan)
            y = symm_mem.empty(len(self.plan) * rmax, n, dtype=dtype, device=device)
            group = self.group or dist.group.WORLD
            h = symm_mem.rendezvous(y, group)
            ptrs = push_targets(h.buffer_ptrs, self.plan, self.rank, n, y.element_size())
            self._symm[key] = (y, h, torch.tensor(ptrs, dtype=torch.int64, device=device))
        return self._symm[key]

    def __call__(self, x, split_k: int = 0, out_dtype=None):
        import torch

        from . import spmm, spmm_push
        if self.push:
            dtype = out_dtype or torch.float32
            y, h, peers = self._push_buffer(x.shape[1], dtype, x.device)
            h.barrier(channel=0)  # every rank is done reading the previous result
            if self.local is not None:
                spmm_push(self.local, x, peers, split_k=split_k, out_dtype=dtype)
            h.barrier(channel=0)  # every rank's rows have landed in every buffer
            if all(sh.rows == max_rows(self.plan) for sh in self.plan):
                return y
            rmax = max_rows(self.plan)
            return torch.cat([y[sh.rank * rmax: sh.rank * rmax + sh.rows] for sh in self.plan], dim=0)
        if self.local is not None:
            y = spmm(self.local, x, split_k=split_k, out_dtype=out_dtype)
        else:
            y = torch.empty((0, x.shape[1]), dtype=out_dtype or torch.float32, device=x.device)
        return allgather_rows(y, self.plan, self.group, comm=self.comm)
