"""GPU prune_magnitude, bit-exact with the reference's
prune_magnitude (proj/src/matrix.cpp:69-100): the KATs of proj/tests/test_matrix.cpp:54-104
and random / heavy-tie / special-value inputs against the CPU oracle port (which the
oracle tests pin to the reference)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gpu_prune(a, beta, inplace=False):
    import torch

    import paper_2309_10285_b200 as tc
    d = torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()
    out = tc.prune_magnitude(d, beta, out=d if inplace else None)
    return out.cpu().numpy().view(np.uint16)


def h(v):
    return np.float16(v).view(np.uint16)


def test_reference_kats():
    a = np.array([[h(1.0), h(-4.0)], [h(2.0), h(3.0)]], np.uint16)  # worked example
    assert _gpu_prune(a, 0.5).tolist() == [[0, 0xC400], [0, 0x4200]]
    a = np.array([[h(2.0)] * 4], np.uint16)  # ties: the larger index goes first
    assert _gpu_prune(a, 0.5).tolist() == [[0x4000, 0x4000, 0, 0]]
    a = np.array([[h(1.0), h(-2.0), h(3.0), h(-4.0)]], np.uint16)
    assert (_gpu_prune(a, 0.0) == a).all() and (_gpu_prune(a, 0.24) == a).all()
    assert (_gpu_prune(a, 1.0) == 0).all()
    a = np.array([[0x7E00, h(1.0), h(2.0), h(3.0)]], np.uint16)  # NaN ranks above every number
    p = _gpu_prune(a, 0.5)
    assert p[0, 0] == 0x7E00 and p[0, 1] == 0 and p[0, 2] == 0 and p[0, 3] == 0x4200


def test_invalid_beta():
    import torch

    import paper_2309_10285_b200 as tc
    d = torch.zeros((4, 4), dtype=torch.float16, device="cuda")
    for beta in (-0.1, 1.5, float("nan")):
        with pytest.raises(tc.TcslError, match="invalid_argument"):
            tc.prune_magnitude(d, beta)


@pytest.mark.parametrize("beta", [0.25, 0.5, 0.8])
def test_heavy_ties_idempotent_and_exact(port, beta):
    rng = np.random.default_rng(42)
    pool = np.array([h(0.0), 0x8000, h(1.0), h(-1.0), h(2.0), h(-2.0), h(0.5)], np.uint16)
    a = pool[rng.integers(0, len(pool), (17, 23))]
    once = _gpu_prune(a, beta)
    assert (once == port.prune_magnitude(a, beta)).all()
    assert (_gpu_prune(once, beta) == once).all()


@pytest.mark.parametrize("shape,beta,seed", [((1, 1), 0.7, 1), ((3, 1001), 0.5, 2), ((300, 517), 0.8, 3),
                                             ((1024, 4096), 0.9, 4), ((2048, 2048), 0.7, 5)])
def test_random_vs_oracle(port, shape, beta, seed):
    a = port.gen_random_sparse(shape[0], shape[1], 0.3, seed)
    want = port.prune_magnitude(a, beta)
    assert (_gpu_prune(a, beta) == want).all()
    assert (_gpu_prune(a, beta, inplace=True) == want).all()


def test_special_values_vs_oracle(port):
    rng = np.random.default_rng(9)
    a = rng.integers(0, 1 << 16, (513, 257), dtype=np.uint32).astype(np.uint16)  # every class: NaN, inf, subnormals
    a[::7, ::5] = 0x7C00
    a[::11, ::3] = 0xFC00
    a[::13, ::2] = 0x8000
    for beta in (0.1, 0.5, 0.93, 1.0):
        assert (_gpu_prune(a, beta) == port.prune_magnitude(a, beta)).all(), beta


def test_large_dense_weight(port):
    """A dense 4096 x 4096 weight (gen_random_sparse at beta=0: many magnitude ties)
    pruned to 80 %: exact against the oracle, and exactly floor(0.8 n) zeros."""
    a = port.gen_random_sparse(4096, 4096, 0.0, 11)
    want = port.prune_magnitude(a, 0.8)
    got = _gpu_prune(a, 0.8)
    assert (got == want).all()
    assert int(((got & 0x7FFF) == 0).sum()) == int(np.floor(0.8 * a.size))
