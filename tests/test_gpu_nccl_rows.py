"""The C-ABI NCCL all-gather of row-sharded Y (tcsl_cuda_allgather_rows)
on the one GPU a test box has: a world-size-1 communicator created through the C-ABI
(unique id, comm init), fp32 and binary16 rows, and the RowShardedSpmm path end to end.
The multi-rank host logic is covered by tests/test_sharding_gloo.py (gloo, CPU)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_nccl_allgather_rows_world1(port):
    import torch

    import paper_2309_10285_b200 as tc
    from paper_2309_10285_b200.sharding import RowShardedSpmm
    assert tc.lib().tcsl_cuda_nccl_available() == 1
    comm = tc.RowComm(0, 1)
    try:
        y = torch.randn((768, 24), device="cuda")
        full = torch.empty_like(y)
        comm.allgather_rows(y, full)
        torch.cuda.synchronize()
        assert torch.equal(full, y)
        h = y.half()
        fh = torch.empty_like(h)
        comm.allgather_rows(h, fh)
        torch.cuda.synchronize()
        assert torch.equal(fh, h)
        a = port.gen_random_sparse(1024, 512, 0.8, 5)
        x = port.gen_random_sparse(512, 32, 0.0, 6)
        t = tc.encode(torch.from_numpy(a.view(np.int16)).cuda())
        xd = torch.from_numpy(x.view(np.int16)).cuda()
        rs = RowShardedSpmm(t, 1, 0, comm=comm)
        got = rs(xd, split_k=1)
        assert torch.equal(got, tc.spmm(t, xd, split_k=1))
    finally:
        comm.close()
