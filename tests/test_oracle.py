"""Pins the C restatement (oracle/tcsl_oracle.c) before anything trusts it.

Mirrors the reference's own hot-path tests: proj/tests/test_codec.cpp,
test_engine.cpp, test_gemm.cpp and acceptance criteria 1-2
(proj/tests/acceptance.cpp:89-185), plus the committed golden fixtures.
"""
import json
import os

import numpy as np
import pytest

from oracle import OracleError, Tcsl

GOLD = os.path.join(os.path.dirname(__file__), "golden")
GOLDEN = [("golden_a.tcsl", 128, 64, 0.3, 11, True, 0xa57f18792a5f0447),
          ("golden_b.tcsl", 256, 128, 0.8, 22, True, 0x2a290613b42e2457),
          ("golden_c.tcsl", 130, 70, 0.5, 33, False, 0xf68ef9afd7dea93a)]


def h(v: float) -> int:
    return int(np.float16(v).view(np.uint16))


@pytest.mark.parametrize("g", GOLDEN, ids=[g[0] for g in GOLDEN])
def test_golden_hashes(port, g):
    name, r, c, beta, seed, reorder, want = g
    a = port.gen_random_sparse(r, c, beta, seed)
    data = port.serialize(port.encode(a, reorder=reorder))
    assert port.fnv1a(data) == want
    with open(os.path.join(GOLD, name), "rb") as f:
        fixture = f.read()
    assert fixture == data
    t = port.deserialize(fixture)
    assert (port.decode(t) == a).all()


def test_kats_fixture(port):
    with open(os.path.join(GOLD, "kats.json")) as f:
        kats = json.load(f)
    for c in kats["encode"]:
        a = port.gen_random_sparse(c["rows"], c["cols"], c["beta"], c["seed"])
        t = port.encode(a, c["m_tb"], c["k_tb"], c["reorder"])
        data = port.serialize(t)
        assert len(t.entries) == c["n_entries"]
        assert hex(port.fnv1a(data)) == c["fnv"], c
    for c in kats["spmm"]:
        a = port.gen_random_sparse(c["m"], c["k"], c["beta"], c["seed_a"])
        b = port.gen_random_sparse(c["k"], c["n"], 0.0, c["seed_b"])
        y = port.spmm(port.encode(a), b, nthreads=4)
        assert hex(port.fnv1a(y.tobytes())) == c["y_fnv"], c


def test_bank_and_entry_layout(port):  # test_codec.cpp:26-46
    a = np.zeros((128, 64), np.uint16)
    a[1, 2] = 0x3C00
    t = port.encode(a)
    assert t.entries[0] == 0x3C000042


def test_encode_worked_example(port):  # test_codec.cpp:48-64
    a = np.zeros((128, 64), np.uint16)
    a[0, 0] = h(1.0)
    a[1, 2] = h(2.0)
    t = port.encode(a)
    assert list(t.offsets) == [0, 32]
    assert t.entries[0] == 0x3C000000 and t.entries[1] == 0x40000042
    for i in range(2, 32):
        assert t.entries[i] >> 16 == 0 and (t.entries[i] & 0xFFFF) == i - 1
    assert (port.decode(t) == a).all()


def test_reorder_greedy_order(port):  # test_codec.cpp:66-84
    a = np.zeros((128, 64), np.uint16)
    a[0, 0], a[1, 0], a[1, 1] = h(1.0), h(2.0), h(3.0)
    nat = port.encode(a, reorder=False)
    assert [e & 0xFFFF for e in nat.entries[:3]] == [0, 64, 65]
    reo = port.encode(a, reorder=True)
    assert [e & 0xFFFF for e in reo.entries[:3]] == [64, 0, 65]


def test_empty_and_dense_tiles(port):  # test_codec.cpp:86-96
    assert list(port.encode(np.zeros((128, 64), np.uint16)).offsets) == [0, 0]
    dense = port.gen_random_sparse(128, 64, 0.0, 17)
    t = port.encode(dense)
    assert list(t.offsets) == [0, 8192]
    assert (port.decode(t) == dense).all()


def test_round_trip_with_negative_zero(port):  # test_codec.cpp:98-117
    rng = np.random.default_rng(88)
    for it in range(12):
        m, k = int(rng.integers(1, 301)), int(rng.integers(1, 151))
        beta = int(rng.integers(0, 1001)) / 1000
        a = port.gen_random_sparse(m, k, beta, int(rng.integers(0, 2**63)))
        if a.size > 3:
            a.reshape(-1)[2] = 0x8000
        t = port.encode(a, reorder=it % 2 == 0)
        want = a.copy()
        want[(want & 0x7FFF) == 0] = 0
        assert (port.decode(t) == want).all()
        assert all((t.offsets[1:] - t.offsets[:-1]) % 32 == 0)


def test_deserialize_rejects_malformed(port):  # test_codec.cpp:182-240
    t = port.encode(port.gen_random_sparse(130, 70, 0.5, 9))
    good = bytearray(port.serialize(t))

    def code(buf):
        with pytest.raises(OracleError) as e:
            port.deserialize(bytes(buf))
        return e.value.errc

    m = good.copy(); m[0] = ord("Y"); assert code(m) == "bad_magic"
    m = good.copy(); m[4] = 2; assert code(m) == "bad_version"
    m = good.copy(); m[7] = 0x80; assert code(m) == "bad_version"
    m = good.copy(); m[8:12] = b"\0\0\0\0"; assert code(m) == "bad_header"
    m = good.copy(); m[20] = 60; assert code(m) == "bad_header"
    m = good.copy(); m[24] ^= 0xFF; assert code(m) == "bad_header"
    m = good.copy(); m[32] = 1; assert code(m) == "inconsistent_offsets"
    m = good.copy(); m[32:36] = b"\xff\xff\xff\xff"; assert code(m) == "inconsistent_offsets"
    assert code(good[:28 + 20 + 2]) == "truncated"
    assert code(good[:10]) == "truncated"
    assert code(good + b"\0") == "trailing_data"


def test_decode_rejects_bad_locations(port):  # test_codec.cpp:242-267
    a = np.zeros((128, 64), np.uint16)
    a[0, 0] = h(1.0)
    t = port.encode(a)
    bad = Tcsl(**{**t.__dict__, "entries": t.entries.copy()})
    bad.entries[1] = 8192
    with pytest.raises(OracleError, match="location_out_of_range"):
        port.decode(bad)
    f = port.gen_random_sparse(100, 64, 0.501, 3)
    tf = port.encode(f)
    i = int(np.nonzero((tf.entries >> 16) == 0)[0][0])
    tf.entries[i] = (0x3C00 << 16) | (110 * 64)
    with pytest.raises(OracleError, match="location_out_of_range"):
        port.decode(tf)


def test_invalid_inputs(port):  # test_codec.cpp:269-273
    with pytest.raises(OracleError, match="invalid_argument"):
        port.encode(np.zeros((0, 0), np.uint16))
    with pytest.raises(OracleError, match="invalid_argument"):
        port.encode(port.gen_random_sparse(16, 16, 0.5, 2), 12, 8)


def test_extract_tile_kat(port):  # test_engine.cpp:21-39
    a = np.zeros((128, 64), np.uint16)
    a[0, 0], a[1, 2], a[127, 63] = h(1.0), h(2.0), h(-3.0)
    buf = port.extract_tile(port.encode(a), 0)
    assert buf[0] == 0x3C00 and buf[66] == 0x4000 and buf[127 * 64 + 63] == 0xC200
    assert int(((buf & 0x7FFF) != 0).sum()) == 3


def test_spmm_bit_exact_small_tiles(port):  # test_engine.cpp:64-85
    rng = np.random.default_rng(77)
    for it in range(25):
        m, k, n = (int(rng.integers(1, 51)), int(rng.integers(1, 41)), int(rng.integers(1, 13)))
        beta = int(rng.integers(0, 1001)) / 1000
        a = port.gen_random_sparse(m, k, beta, int(rng.integers(0, 2**63)))
        b = port.gen_random_sparse(k, n, 0.1, int(rng.integers(0, 2**63)))
        t = port.encode(a, 16, 8, it % 2 == 0)
        got = port.spmm(t, b)
        want = port.dense_gemm(port.decode(t), b, 16, 8)
        assert got.tobytes() == want.tobytes()


def test_reg_pressure_kat(port):  # test_engine.cpp:101-113
    dense = port.gen_random_sparse(128, 64, 0.0, 3)
    assert port.reg_pressure(port.encode(dense)) == 64
    assert port.reg_pressure(port.encode(port.prune_magnitude(dense, 0.8))) == 13
    assert port.reg_pressure(port.encode(dense), 96) == 86


def test_gemm_order_and_signed_zero(port):  # test_gemm.cpp:89-117
    a = np.array([[h(4096), h(1), h(-4096)]], np.uint16)
    b = np.array([[h(4096)], [h(1)], [h(4096)]], np.uint16)
    c = port.dense_gemm(a, b, 16, 8)
    assert c.view(np.uint32)[0, 0] == 0
    a = np.array([[0x8000, 0x0000]], np.uint16)
    b = np.array([[h(3)], [h(-5)]], np.uint16)
    assert port.dense_gemm(a, b, 16, 8).view(np.uint32)[0, 0] == 0


def test_half_conversions(port):  # test_half.cpp:68-87 (exhaustive widening)
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    want = bits.view(np.float16).astype(np.float32)
    got = np.array([port.f32_from_f16(int(b)) for b in bits[::97]], np.float32)
    ref = want[::97]
    same = (got.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(got) & np.isnan(ref))
    assert same.all()
    assert port.f16_from_f32(float("nan")) == 0x7E00
    assert port.f16_from_f32(65520.0) == 0x7C00


def test_port_matches_reference(port, ref):  # acceptance.cpp:89-120, reduced
    rng = np.random.default_rng(20240817)
    ns = [8, 16, 32, 64]
    for i in range(30):
        m = 128 * int(rng.integers(1, 5)) if i < 20 else int(rng.integers(1, 701))
        k = 64 * int(rng.integers(1, 8)) if i < 20 else int(rng.integers(1, 701))
        n = ns[i % 4]
        beta = [0.0, 0.5, 0.7, 0.8, 0.9][i % 5]
        sa, sb = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**63))
        a = ref.gen_random_sparse(m, k, beta, sa)
        assert (a == port.gen_random_sparse(m, k, beta, sa)).all()
        b = ref.gen_random_sparse(k, n, 0.05, sb)
        tr = ref.encode(a, reorder=i % 2 == 0)
        tp = port.encode(a, reorder=i % 2 == 0)
        assert (tr.offsets == tp.offsets).all() and (tr.entries == tp.entries).all()
        assert ref.spmm(tr, b).tobytes() == port.spmm(tp, b).tobytes()
        assert ref.spmm(tr, b, 3).tobytes() == port.spmm(tp, b, 2).tobytes()
