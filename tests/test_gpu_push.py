"""The all-gather fused into the SpMM epilogue (tcsl_cuda_spmm_push, SURVEY.md §8e /
BASELINE configs[4]) on the one GPU a test box has: the kernel stores every finished
Y row block into n_peers destinations, here separate local buffers standing in for
peers' symmetric-memory Y, each checked bit for bit against the ordinary spmm (same
kernel math) — split-K 1 and 3 (the K3 pass pushes), fp32 and binary16 with
bias + activation, the exact path — and a world-size-1 symmetric-memory run of
RowShardedSpmm(push=True). Multi-rank host logic: tests/test_sharding_gloo.py."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()


@pytest.mark.parametrize("split,f16,act,exact", [(1, False, None, False), (3, False, None, False),
                                                 (1, True, "relu", False), (2, True, "gelu_tanh", False),
                                                 (1, False, None, True)])
def test_push_matches_spmm(port, split, f16, act, exact):
    import torch

    import paper_2309_10285_b200 as tc
    m, k, n = 1000, 1536, 24
    a = port.gen_random_sparse(m, k, 0.85, 3)
    x = _dev(port.gen_random_sparse(k, n, 0.0, 4))
    t = tc.encode(_dev(a))
    dt = torch.float16 if f16 else torch.float32
    bias = torch.randn(m, device="cuda") if act else None
    want = tc.spmm(t, x, split_k=split, exact=exact, bias=bias, activation=act, out_dtype=dt)
    # three "peers": full-Y buffers of 3 * 1024 rows; this shard is rank 1 (rows 1024..)
    bufs = [torch.full((3 * 1024, n), 7.0, dtype=dt, device="cuda") for _ in range(3)]
    from paper_2309_10285_b200.sharding import Shard, push_targets
    plan = [Shard(r, 8 * r, 8 * r + 8, 1024 * r, 1024 if r < 2 else 1000) for r in range(3)]
    ptrs = push_targets([b.data_ptr() for b in bufs], plan, 1, n, bufs[0].element_size())
    tc.spmm_push(t, x, torch.tensor(ptrs, dtype=torch.int64, device="cuda"), split_k=split, exact=exact, bias=bias,
                 activation=act, out_dtype=dt)
    torch.cuda.synchronize()
    for b in bufs:
        assert torch.equal(b[1024:1024 + m], want)
        assert (b[:1024] == 7.0).all() and (b[1024 + m:] == 7.0).all()  # nothing outside the shard's rows


def test_push_argument_errors(port):
    import torch

    import paper_2309_10285_b200 as tc
    a = port.gen_random_sparse(256, 128, 0.8, 1)
    t = tc.encode(_dev(a))
    x = _dev(port.gen_random_sparse(128, 8, 0.0, 2))
    with pytest.raises(tc.TcslError, match="invalid_argument"):
        tc.spmm_push(t, x, torch.zeros(0, dtype=torch.int64, device="cuda"))
    with pytest.raises(tc.TcslError, match="invalid_argument"):
        tc.spmm_push(t, x, torch.zeros(2, dtype=torch.int32, device="cuda"))


def test_row_sharded_push_symmetric_memory_world1(port):
    """RowShardedSpmm(push=True) end to end on a world-size-1 NCCL group: symmetric-memory
    Y, pushed epilogue, device barriers; equals the plain SpMM."""
    import torch
    import torch.distributed as dist

    import paper_2309_10285_b200 as tc
    from paper_2309_10285_b200.sharding import RowShardedSpmm
    try:
        import torch.distributed._symmetric_memory  # noqa: F401
    except ImportError as e:
        pytest.skip(f"no symmetric memory in this torch: {e}")
    own = not dist.is_initialized()
    if own:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29600 + os.getpid() % 1000))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        a = port.gen_random_sparse(768, 1024, 0.8, 7)
        x = _dev(port.gen_random_sparse(1024, 32, 0.0, 8))
        t = tc.encode(_dev(a))
        want = tc.spmm(t, x)
        rs = RowShardedSpmm(t, 1, 0, push=True)
        for _ in range(2):  # the buffer is reused across calls
            y = rs(x)
            torch.cuda.synchronize()
            assert torch.equal(y, want)
    finally:
        if own:
            dist.destroy_process_group()
