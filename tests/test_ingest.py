"""TCSL container ingest + device-side structural validation.

CPU: tcsl_cuda_parse_header (host code) reports deserialize_tcsl's error classes for
header-level damage (proj/tests/test_codec.cpp:182-240, proj/src/tcsl_format.cpp:180-222).
GPU: tcsl_cuda_ingest uploads and validates offsets + entries on the device; the
error classes and the decoded matrix equal the oracle's deserialize + decode, and
entry-level anomalies (repeated locations, fringe payloads, out-of-range locations)
come back as flags. Repeated locations decode last-writer-wins like the reference."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2309_10285_b200 as tc
from oracle import OracleError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _good(port):
    a = port.gen_random_sparse(130, 70, 0.5, 9)
    t = port.encode(a)
    assert t.num_tiles == 4
    return a, bytearray(port.serialize(t))


def _mutations(good):
    offsets_at, entries_at = 28, 28 + 4 * 5
    out = []

    def mut(label, f):
        b = bytearray(good)
        f(b)
        out.append((label, bytes(b)))

    mut("magic", lambda b: b.__setitem__(0, ord("Y")))
    mut("version", lambda b: b.__setitem__(4, 2))
    mut("flags", lambda b: b.__setitem__(7, 0x80))
    mut("zero rows", lambda b: b.__setitem__(slice(8, 12), b"\0\0\0\0"))
    mut("tile dims", lambda b: b.__setitem__(20, 60))
    mut("num_tiles", lambda b: b.__setitem__(24, b[24] ^ 0xFF))
    mut("group quantum", lambda b: b.__setitem__(offsets_at + 4, 1))
    mut("monotonicity", lambda b: b.__setitem__(slice(offsets_at + 4, offsets_at + 8), b"\xff" * 4))
    mut("entry payload cut", lambda b: b.__delitem__(slice(entries_at + 2, None)))
    mut("header cut", lambda b: b.__delitem__(slice(10, None)))
    mut("trailing byte", lambda b: b.append(0))
    mut("last offset too large", lambda b: b.__setitem__(slice(offsets_at + 16, offsets_at + 20),
                                                         (int.from_bytes(b[offsets_at + 16:offsets_at + 20], "little")
                                                          + 32).to_bytes(4, "little")))
    return out


def _parse(data: bytes) -> int:
    h = tc.Header()
    arr = np.frombuffer(data, np.uint8)
    return tc.lib().tcsl_cuda_parse_header(C.c_void_p(arr.ctypes.data) if arr.size else None, arr.size, C.byref(h))


def _oracle_status(port, data: bytes) -> int:
    try:
        port.deserialize(data)
        return 0
    except OracleError as e:
        return e.status


def test_parse_header_error_classes_cpu(port):
    _, good = _good(port)
    assert _parse(bytes(good)) == 0
    for label, data in _mutations(good):
        want = _oracle_status(port, data)
        got = _parse(data)
        if label in ("group quantum", "monotonicity"):
            # sizes still consistent: the offset table is validated on the device (tcsl_cuda_ingest)
            assert got == 0 and want == 7, label
        else:
            assert got == want, (label, got, want)


@pytest.mark.gpu
def test_ingest_golden_files(port):
    for name in ("golden_a.tcsl", "golden_b.tcsl", "golden_c.tcsl"):
        path = os.path.join(GOLD, name)
        t = tc.load_tcsl(path)
        want = port.deserialize(open(path, "rb").read())
        off, ent = t.to_host()
        assert (off == want.offsets).all() and (ent == want.entries).all()
        assert (t.m, t.k, t.reordered) == (want.m, want.k, want.reordered)
        assert t.tc_ready and t.ingest_flags == 0
        assert tc.serialize_tcsl(t) == open(path, "rb").read()
        assert (tc.decode(t).cpu().numpy().view(np.uint16) == port.decode(want)).all()


@pytest.mark.gpu
def test_ingest_error_classes(port):
    _, good = _good(port)
    for label, data in _mutations(good):
        want = _oracle_status(port, data)
        if want == 0:
            continue
        with pytest.raises(tc.TcslError) as ei:
            tc.load_tcsl(data)
        assert ei.value.status == want, label


@pytest.mark.gpu
def test_ingest_large_pageable_staged(port):
    # a 4096 x 2048 matrix: entries > the 8 MiB staging buffer, so the double-buffered path runs
    a = port.gen_random_sparse(4096, 2048, 0.5, 5)
    t0 = port.encode(a)
    data = port.serialize(t0)
    assert len(data) > 8 << 20
    t = tc.load_tcsl(data)
    off, ent = t.to_host()
    assert (off == t0.offsets).all() and (ent == t0.entries).all()


def _dev_matrix(t):
    return tc.TcslMatrix.from_host(t.m, t.k, t.offsets, t.entries, tc.TileConfig(t.m_tb, t.k_tb), t.reordered)


@pytest.mark.gpu
def test_validate_entries_flags_and_classes(port):
    import torch
    a = np.zeros((128, 64), np.uint16)
    a[0, 0] = 0x3C00
    t = port.encode(a)
    assert tc.check_entries(_dev_matrix(t)) == 0
    bad = port.encode(a)
    bad.entries[1] = 8192  # past the tile (test_codec.cpp:242-250)
    with pytest.raises(tc.TcslError, match="location_out_of_range"):
        tc.check_entries(_dev_matrix(bad), tc.CHECK_DECODE)
    with pytest.raises(tc.TcslError, match="location_out_of_range"):
        tc.check_entries(_dev_matrix(bad), tc.CHECK_SPMM)
    assert tc.check_entries(_dev_matrix(bad), tc.CHECK_INGEST) & tc.FLAG_LOCATION_RANGE
    # fringe payload (test_codec.cpp:252-262): row 110 of a 100-row matrix
    f = port.gen_random_sparse(100, 64, 0.501, 3)
    tf = port.encode(f)
    i = int(np.nonzero((tf.entries >> 16) == 0)[0][0])
    tf.entries[i] = (0x3C00 << 16) | (110 * 64)
    with pytest.raises(tc.TcslError, match="location_out_of_range"):
        tc.check_entries(_dev_matrix(tf), tc.CHECK_DECODE)
    assert tc.check_entries(_dev_matrix(tf), tc.CHECK_SPMM) & tc.FLAG_FRINGE_PAYLOAD
    # inconsistent offsets wins over location errors (the reference checks offsets first)
    both = port.encode(a)
    both.entries[1] = 8192
    both.offsets = np.array([0, 16], np.uint32)
    with pytest.raises(tc.TcslError, match="inconsistent_offsets"):
        tc.check_entries(_dev_matrix(both), tc.CHECK_DECODE)
    del torch


@pytest.mark.gpu
def test_repeated_locations_last_writer_wins(port):
    """A location repeated inside a tile: the reference's decode / extract_tile keep
    the last entry (tcsl_format.cpp:137-152, engine.cpp:17-22). GPU decode and spmm
    (which routes such matrices to the exact path) must agree bit for bit, every run."""
    import torch
    a = port.gen_random_sparse(256, 128, 0.7, 21)
    t = port.encode(a)
    rng = np.random.default_rng(3)
    ent = t.entries.copy()
    # in tile 0 and tile 3, copy the locations of some entries onto later entries with new values
    for tile in (0, 3):
        lo, hi = int(t.offsets[tile]), int(t.offsets[tile + 1])
        for _ in range(40):
            i, j = sorted(rng.choice(np.arange(lo, hi), 2, replace=False))
            ent[j] = (ent[j] & 0xFFFF0000) | (ent[i] & 0xFFFF)
    t.entries = ent
    want = port.decode(t)
    x = port.gen_random_sparse(128, 16, 0.0, 4)
    want_y = port.spmm(t, x)
    d = _dev_matrix(t)
    assert tc.check_entries(d, tc.CHECK_SPMM) & tc.FLAG_DUPLICATE_LOCATIONS
    for _ in range(3):
        assert (tc.decode(d).cpu().numpy().view(np.uint16) == want).all()
        d2 = _dev_matrix(t)
        y = tc.spmm(d2, torch.from_numpy(x.view(np.int16)).cuda()).cpu().numpy()
        assert d2.tc_ready is False
        assert y.tobytes() == want_y.tobytes()


@pytest.mark.gpu
def test_partial_groups_accepted_like_reference(port):
    """Spans that are not whole groups are legal for the reference's spmm
    (engine.cpp:8-14 checks only each tile's own span): same bits as the oracle."""
    import torch
    a = port.gen_random_sparse(256, 128, 0.8, 8)
    t = port.encode(a)
    t.offsets = t.offsets.copy()
    t.offsets[1] += 16  # tile 0 takes 16 entries of tile 1
    x = port.gen_random_sparse(128, 8, 0.0, 2)
    want = port.spmm(t, x)
    y = tc.spmm(_dev_matrix(t), torch.from_numpy(x.view(np.int16)).cuda()).cpu().numpy()
    assert y.tobytes() == want.tobytes()
    t.offsets[1] = t.entries.size + 32  # past the entries: inconsistent_offsets
    with pytest.raises(tc.TcslError, match="inconsistent_offsets"):
        tc.spmm(_dev_matrix(t), torch.from_numpy(x.view(np.int16)).cuda())
