"""The a-priori B200 time model (tcsl_cuda_spmm_estimate), the B200 counterpart of the
reference's estimate_time (proj/src/pipeline.cpp:214-273). Host only: runs on CPU.
Pinned to the committed B200 measurement of all 84 bench cells."""
import json
import os

import numpy as np
import pytest

import paper_2309_10285_b200 as tc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_model_matches_measured_cells():
    with open(os.path.join(ROOT, "profiles", "r02_bench_v3.json")) as f:
        cells = json.load(f)["cells"]
    err = []
    for c in cells:
        e = tc.estimate(c["M"], c["K"], c["N"], c["E"], c["split"])
        assert e["split"] == c["split"]
        err.append(abs(e["us"] - c["us"]) / c["us"])
    assert np.median(err) <= 0.03 and max(err) <= 0.2, (np.median(err), max(err))


def test_model_terms():
    # OPT-66B FFN1 at 80 % (SURVEY Appendix B's E): HBM term = algorithmic bytes / peak
    m, k, n, E = 36864, 9216, 16, 68590112
    e = tc.estimate(m, k, n, E, 1, hbm_gbs=8000.0)
    T = (m // 128) * (k // 64)
    assert e["hbm_us"] == pytest.approx((4 * E + 4 * (T + 1) + 2 * k * n + 4 * m * n) / 8e6)
    assert e["us"] == pytest.approx(e["fixed_us"] + max(e["hbm_us"], e["tensor_us"], e["smem_us"], e["chain_us"]))
    assert e["bound"] == "chain"  # the measured limiter (measured limiters)
    # denser -> slower; more columns -> not faster
    assert tc.estimate(m, k, n, 2 * E)["us"] > tc.estimate(m, k, n, E)["us"]
    assert tc.estimate(m, k, 64, E)["us"] >= tc.estimate(m, k, 8, E)["us"]
    # split-K adds the reduction pass
    assert tc.estimate(9216, 36864, 8, 34615808, 2)["fixed_us"] > tc.estimate(9216, 36864, 8, 34615808, 1)["fixed_us"]
    with pytest.raises(tc.TcslError, match="invalid_argument"):
        tc.estimate(0, k, n, E)
