"""Multi-process (world_size 2 and 3, gloo, CPU) check of the row-sharding path:
each rank slices its shard of the Tiled-CSL matrix, computes its rows of Y
with the CPU oracle (standing in for the GPU kernel, which runs per shard in
tests/test_gpu_spmm.py::test_sharded_rows_match_full), and the all-gather
assembles the full Y — bit-identical to the unsharded oracle result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_10285_b200.sharding import allgather_rows, shard_plan, slice_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, k, n, beta, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from oracle import Tcsl
    P = oracle.port()
    a = P.gen_random_sparse(m, k, beta, 11)
    x = P.gen_random_sparse(k, n, 0.0, 12)
    t = P.encode(a)
    plan = shard_plan(m, 128, world)
    sh = plan[rank]
    off, ent = slice_rows(t.offsets, t.entries, t.tiles_k, sh)
    if sh.rows:
        ts = Tcsl(sh.rows, k, 128, 64, True, off, ent)
        # the slice is exactly encode() of those rows
        re = P.encode(a[sh.row0: sh.row0 + sh.rows])
        assert (re.offsets == off).all() and (re.entries == ent).all()
        y_local = torch.from_numpy(P.spmm(ts, x))
    else:
        y_local = torch.zeros((0, n), dtype=torch.float32)
    y = allgather_rows(y_local, plan)
    if rank == 0:
        np.save(out_path, y.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(2, 1000), (3, 700), (2, 100)])
def test_row_sharded_allgather_matches_full(tmp_path, world, m):
    k, n, beta = 300, 16, 0.8
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(world, _free_port(), m, k, n, beta, out), nprocs=world, join=True)
    import oracle
    P = oracle.port()
    a = P.gen_random_sparse(m, k, beta, 11)
    x = P.gen_random_sparse(k, n, 0.0, 12)
    want = P.spmm(P.encode(a), x)
    got = np.load(out)
    assert got.shape == want.shape
    assert got.tobytes() == want.tobytes()


def test_shard_plan_covers_rows():
    for m in (1, 127, 128, 129, 49152, 12345):
        for world in (1, 2, 3, 4, 8):
            plan = shard_plan(m, 128, world)
            assert sum(s.rows for s in plan) == m
            assert all(s.row0 == s.tr0 * 128 for s in plan)
            assert [s.tr1 for s in plan[:-1]] == [s.tr0 for s in plan[1:]]


@pytest.mark.parametrize("world,m", [(2, 49152), (8, 49152), (3, 1000), (4, 300)])
def test_push_targets_tile_the_buffer(world, m):
    """Fused all-gather addressing (sharding.push_targets): rank r's rows land at
    r * rmax rows into every rank's full-Y buffer; over all ranks the written row
    ranges are disjoint, in rank order, and cover every real row once."""
    from paper_2309_10285_b200.sharding import max_rows, push_targets
    plan = shard_plan(m, 128, world)
    n, eb = 32, 4
    bases = [1 << 40, 2 << 40, 3 << 40][:1] * world
    rmax = max_rows(plan)
    covered = []
    for sh in plan:
        t = push_targets([bases[0]] * world, plan, sh.rank, n, eb)
        assert len(t) == world and len(set(t)) == 1
        row0 = (t[0] - bases[0]) // (n * eb)
        assert row0 == sh.rank * rmax
        covered.append((row0, row0 + sh.rows))
    for (a0, a1), (b0, b1) in zip(covered, covered[1:]):
        assert a1 <= b0
    assert sum(b - a for a, b in covered) == m
