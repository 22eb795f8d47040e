"""CPU checks of bench.py's measurement contract (no GPU): the cell set is
BASELINE.json configs[1] (48 OPT-66B SpMMs), the algorithmic bytes follow
SURVEY.md §8d (4E + 4(T+1) + 2KN + 4MN), and the roofline traffic comes from a
committed ncu summary of the reference cell."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(**kw):
    a = argparse.Namespace(only="", suite="opt66b", split=0)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_default_cells_are_configs1():
    cells = bench.cell_list(_args())
    assert len(cells) == 48
    assert {c[0] for c in cells} == {"qkv", "out", "ffn1", "ffn2"}
    assert sorted({c[1] for c in cells}) == [0.7, 0.8, 0.9]
    assert sorted({c[2] for c in cells}) == [8, 16, 32, 64]
    assert bench.SHAPES["ffn1"] == (36864, 9216) and bench.SHAPES["ffn2"] == (9216, 36864)


def test_parse_only():
    assert bench.parse_only("ffn2:0.9:8,qkv:0.8:64") == [("ffn2", 0.9, 8), ("qkv", 0.8, 64)]


def test_alg_bytes_formula():
    class T:  # the fields alg_bytes reads from a TcslMatrix
        m, k, n_entries, num_tiles = 256, 128, 3200, 4  # 2 x 2 tiles of 128 x 64
    t = T()
    tiles = 2 * 2
    want = 4 * 3200 + 4 * (tiles + 1) + 2 * 128 * 16 + 4 * 256 * 16
    assert bench.alg_bytes(t, 16) == want


def test_ncu_traffic_uses_reference_cell_summary():
    tr = bench.ncu_traffic()
    assert tr is not None
    assert "beta=0.8 N=16" in tr["cell"] and tr["source"].startswith("profiles/")
    assert 0.98 < tr["dram_bytes_per_launch"] / tr["alg_bytes_per_launch"] < 1.1
