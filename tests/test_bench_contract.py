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
    a = argparse.Namespace(only="", suite="all", split=0)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_default_cells_are_configs1_and_configs3():
    cells = bench.cell_list(_args())
    assert len(cells) == 84
    assert {c[0] for c in cells} == {"qkv", "out", "ffn1", "ffn2", "qkv175", "ffn1_175", "ffn2_175"}
    assert sorted({c[1] for c in cells}) == [0.7, 0.8, 0.9]
    assert sorted({c[2] for c in cells}) == [8, 16, 32, 64]
    assert bench.SHAPES["ffn1"] == (36864, 9216) and bench.SHAPES["ffn2"] == (9216, 36864)
    assert bench.SHAPES["ffn1_175"] == (49152, 12288) and bench.SHAPES["ffn2_175"] == (12288, 49152)


def test_cells_never_reuse_a_weight_while_l2_resident():
    """N is the outer loop: two uses of one compressed weight are separated by all the
    other weights of the step (> 126 MB of L2 many times over)."""
    cells = bench.cell_list(_args())
    last = {}
    for i, (nm, b, n) in enumerate(cells):
        if (nm, b) in last:
            assert i - last[(nm, b)] == len(bench.weight_list(cells))
        last[(nm, b)] = i


def test_host_generator_is_the_reference_generator(port):
    a = bench.gen_random_sparse(300, 200, 0.8, 1)
    assert (a == port.gen_random_sparse(300, 200, 0.8, 1)).all()


def test_both_arms_report_the_same_config():
    assert bench.bench_config(_args(), 1) == bench.bench_config(_args(), 1)
    assert "workload" in bench.bench_config(_args(), 1)


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
