"""GPU encoder / decoder parity: bit-exact against the CPU oracle and the
reference's golden artifacts (proj/tests/acceptance.cpp:60-64, test_codec.cpp)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()


def _gpu_encode(a, m_tb=128, k_tb=64, reorder=True):
    import paper_2309_10285_b200 as tc
    return tc.encode(_dev(a), tc.TileConfig(m_tb, k_tb), reorder)


def _same(port, a, m_tb=128, k_tb=64, reorder=True):
    t = _gpu_encode(a, m_tb, k_tb, reorder)
    off, ent = t.to_host()
    want = port.encode(a, m_tb, k_tb, reorder)
    assert off.shape == want.offsets.shape and (off == want.offsets).all()
    assert ent.shape == want.entries.shape
    bad = np.nonzero(ent != want.entries)[0]
    assert bad.size == 0, f"first mismatch at {bad[:5]}: {ent[bad[:5]]} vs {want.entries[bad[:5]]}"
    return t, want


GOLDEN = [("golden_a.tcsl", 128, 64, 0.3, 11, True, 0xa57f18792a5f0447),
          ("golden_b.tcsl", 256, 128, 0.8, 22, True, 0x2a290613b42e2457),
          ("golden_c.tcsl", 130, 70, 0.5, 33, False, 0xf68ef9afd7dea93a)]


@pytest.mark.parametrize("g", GOLDEN, ids=[g[0] for g in GOLDEN])
def test_golden_artifacts(port, g):
    from oracle import Tcsl
    name, r, c, beta, seed, reorder, want_hash = g
    a = port.gen_random_sparse(r, c, beta, seed)
    t = _gpu_encode(a, reorder=reorder)
    off, ent = t.to_host()
    data = port.serialize(Tcsl(r, c, 128, 64, reorder, off, ent))
    assert port.fnv1a(data) == want_hash
    with open(os.path.join(GOLD, name), "rb") as f:
        assert f.read() == data


def test_kat_fixture(port):
    from oracle import Tcsl
    with open(os.path.join(GOLD, "kats.json")) as f:
        kats = json.load(f)["encode"]
    for c in kats:
        a = port.gen_random_sparse(c["rows"], c["cols"], c["beta"], c["seed"])
        t = _gpu_encode(a, c["m_tb"], c["k_tb"], c["reorder"])
        off, ent = t.to_host()
        data = port.serialize(Tcsl(c["rows"], c["cols"], c["m_tb"], c["k_tb"], c["reorder"], off, ent))
        assert hex(port.fnv1a(data)) == c["fnv"], c


def test_worked_example_and_greedy_order(port):  # test_codec.cpp:48-84
    a = np.zeros((128, 64), np.uint16)
    a[0, 0], a[1, 2] = 0x3C00, 0x4000
    t, _ = _same(port, a)
    _, ent = t.to_host()
    assert ent[0] == 0x3C000000 and ent[1] == 0x40000042
    b = np.zeros((128, 64), np.uint16)
    b[0, 0], b[1, 0], b[1, 1] = 0x3C00, 0x4000, 0x4200
    t, _ = _same(port, b)
    assert [int(e) & 0xFFFF for e in t.to_host()[1][:3]] == [64, 0, 65]
    _same(port, b, reorder=False)
    _same(port, np.zeros((128, 64), np.uint16))


@pytest.mark.parametrize("cfg", [(128, 64), (16, 8), (256, 64), (64, 32), (8, 512), (512, 8), (64, 1024)])
def test_fuzz_tile_configs(port, cfg):
    rng = np.random.default_rng(hash(cfg) & 0xFFFF)
    for it in range(6):
        m, k = int(rng.integers(1, 700)), int(rng.integers(1, 700))
        beta = float(rng.choice([0.0, 0.3, 0.5, 0.7, 0.8, 0.9, 0.99, 1.0]))
        a = port.gen_random_sparse(m, k, beta, int(rng.integers(0, 2**62)))
        _same(port, a, cfg[0], cfg[1], it % 2 == 0)


def test_special_bit_patterns(port):
    rng = np.random.default_rng(5)
    a = rng.integers(0, 65536, size=(300, 190), dtype=np.uint32).astype(np.uint16)
    a[rng.random(a.shape) < 0.6] = 0
    specials = np.array([0x8000, 0x7C00, 0xFC00, 0x7E00, 0x7C01, 0x0001, 0x83FF, 0x03FF], np.uint16)
    idx = rng.integers(0, a.size, 2000)
    a.reshape(-1)[idx] = specials[rng.integers(0, len(specials), 2000)]
    for reorder in (True, False):
        _same(port, a, reorder=reorder)
        _same(port, a, 16, 8, reorder)


def test_c1_full_size_bit_exact(port):  # config 0 shape: 7168 x 7168 at 80 %
    import paper_2309_10285_b200 as tc
    a = port.gen_random_sparse(7168, 7168, 0.8, 1)
    t, want = _same(port, a)
    assert t.n_entries == 10374432  # SURVEY.md Appendix A.6 (seed 1)
    assert port.reg_pressure(want) == 14


def test_decode_round_trip_full_size():
    """encode -> decode is the identity (up to -0 -> +0) at a BASELINE shape."""
    import torch

    import paper_2309_10285_b200 as tc
    w = tc.gen_synthetic(9216, 36864, 0.9, 7)
    w.view(-1)[::1001] = -32768  # -0.0 folds to +0.0
    t = tc.encode(w)
    d = tc.decode(t)
    want = torch.where((w & 0x7FFF) == 0, torch.zeros_like(w), w)
    assert torch.equal(d, want)
    assert all(int(x) % 32 == 0 for x in torch.diff(t.offsets.long()).unique().tolist())


def test_decode_errors(port):
    import paper_2309_10285_b200 as tc
    a = np.zeros((128, 64), np.uint16)
    a[0, 0] = 0x3C00
    t = _gpu_encode(a)
    t.entries[1] = 8192
    with pytest.raises(tc.TcslError, match="location_out_of_range"):
        tc.decode(t)
    f = port.gen_random_sparse(100, 64, 0.501, 3)
    tf = _gpu_encode(f)
    off, ent = tf.to_host()
    i = int(np.nonzero((ent >> 16) == 0)[0][0])
    tf.entries[i] = int(np.int32(np.uint32((0x3C00 << 16) | (110 * 64)).view(np.int32)))
    with pytest.raises(tc.TcslError, match="location_out_of_range"):
        tc.decode(tf)
    t2 = _gpu_encode(a)
    t2.offsets[1] = 16
    with pytest.raises(tc.TcslError, match="inconsistent_offsets"):
        tc.validate(t2)


def test_shard_slices_equal_reencoding(port):
    import paper_2309_10285_b200 as tc
    a = port.gen_random_sparse(1000, 700, 0.8, 11)
    t = _gpu_encode(a)
    for g in (2, 3, 4):
        tm = t.tiles_m
        bounds = [tm * i // g for i in range(g + 1)]
        for tr0, tr1 in zip(bounds[:-1], bounds[1:]):
            sh = tc.shard_rows(t, tr0, tr1)
            off, ent = sh.to_host()
            want = port.encode(a[tr0 * 128:min(1000, tr1 * 128)])
            assert (off == want.offsets).all() and (ent == want.entries).all()


def _fused_same(a, slack=0):
    """The one-pass encoder (tcsl_cuda_encode_fused) gives count+emit's bits."""
    import paper_2309_10285_b200 as tc
    w = _dev(a)
    t = tc.encode(w)
    tf = tc.encode(w, capacity=t.n_entries + slack)
    off, ent = t.to_host()
    offf, entf = tf.to_host()
    assert (off == offf).all() and (ent == entf).all()
    return t


def test_fused_encoder_matches_two_pass(port):
    rng = np.random.default_rng(77)
    for it in range(10):
        m, k = int(rng.integers(1, 900)), int(rng.integers(1, 900))
        beta = float(rng.choice([0.0, 0.5, 0.8, 0.9, 0.99, 1.0]))
        a = port.gen_random_sparse(m, k, beta, int(rng.integers(0, 2**62)))
        t = _fused_same(a, slack=int(rng.integers(0, 100)))
        want = port.encode(a)
        off, ent = t.to_host()
        assert (off == want.offsets).all() and (ent == want.entries).all()


def test_fused_encoder_full_size_and_overflow(port):
    """OPT-66B FFN1 at 80 %: one pass == two passes; a too-small capacity falls back
    to emit with the fused pass's offsets."""
    import torch

    import paper_2309_10285_b200 as tc
    w = tc.gen_synthetic(36864, 9216, 0.8, 3)
    t = tc.encode(w)
    tf = tc.encode(w, capacity=t.n_entries)
    assert torch.equal(t.offsets, tf.offsets) and torch.equal(t.entries, tf.entries)
    small = tc.encode(w, capacity=t.n_entries // 2)
    assert torch.equal(t.offsets, small.offsets) and torch.equal(t.entries, small.entries)


def test_encoder_unaligned_and_odd_widths(port):
    """Fast-path guards: a W view that is not 16-byte aligned, odd k, k % 8 != 0."""
    import paper_2309_10285_b200 as tc
    a = port.gen_random_sparse(300, 513, 0.7, 9)
    big = _dev(a.reshape(-1))
    for (m, k, shift) in [(300, 512, 1), (299, 511, 3), (257, 136, 0), (130, 66, 2)]:
        w = big[shift:shift + m * k].view(m, k)
        t = tc.encode(w)
        want = port.encode(w.cpu().numpy().view(np.uint16))
        off, ent = t.to_host()
        assert (off == want.offsets).all() and (ent == want.entries).all(), (m, k, shift)
        _fused_same(w.cpu().numpy().view(np.uint16))


def test_encoder_extreme_bank_counts(port):
    """Every element nonzero (c_b = 256 for all banks), one bank column only, one row only."""
    rng = np.random.default_rng(3)
    full = rng.integers(1, 0x7BFF, size=(256, 128), dtype=np.uint32).astype(np.uint16)
    _same(port, full)
    col = np.zeros((128, 64), np.uint16)
    col[:, 0::8] = 0x3C00
    _same(port, col)
    row = np.zeros((128, 64), np.uint16)
    row[5, :] = 0x3C00
    row[5, 7] = 0x8000  # -0.0: numerically zero, becomes a pad position candidate
    _same(port, row)
    _fused_same(full)
    _fused_same(col)
    _fused_same(row)
