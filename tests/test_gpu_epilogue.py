"""Fused SpMM epilogue: Y = act(W X + bias), stored as fp32 or
narrowed to binary16 exactly like f16_from_f32 (proj/src/half.cpp:10-40; the CLI's
--out-f16, proj/tools/tcsl_main.cpp:182-186).

Bit-exact on the exact path (the reference's product bits, then one fp32 add, ReLU,
RNE narrowing with canonical NaN); within the north-star tolerance (plus half a binary16
ulp when narrowed) on the tensor-core path, direct epilogue (split 1) and through the
split-K reduction (split > 1)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ELEM = 2.0 ** -10


def _case(port, m, k, n, beta, seed):
    import torch

    import paper_2309_10285_b200 as tc
    a = port.gen_random_sparse(m, k, beta, seed)
    x = port.gen_random_sparse(k, n, 0.0, seed + 1)
    t = tc.encode(torch.from_numpy(a.view(np.int16)).cuda())
    tp = port.encode(a)
    want = port.spmm(tp, x, 8)
    bound = port.spmm(port.encode(a & 0x7FFF), x & 0x7FFF, 8)
    rng = np.random.default_rng(seed)
    bias = (rng.standard_normal(m) * 64).astype(np.float32)
    return t, torch.from_numpy(x.view(np.int16)).cuda(), want, bound, bias


def _np_f16_bits(v32):
    """f16_from_f32 on an array (finite / inf inputs: numpy's RNE cast; NaN -> 0x7E00)."""
    b = v32.astype(np.float16).view(np.uint16).copy()
    b[np.isnan(v32)] = 0x7E00
    return b


def _relu(v):
    return np.where(v > 0, v, np.where(np.isnan(v), v, np.float32(0))).astype(np.float32)


@pytest.mark.parametrize("act", [None, "relu"])
@pytest.mark.parametrize("f16", [False, True])
def test_exact_path_bit_exact(port, act, f16):
    import torch

    import paper_2309_10285_b200 as tc
    t, x, want, _, bias = _case(port, 300, 200, 12, 0.8, 5)
    y = tc.spmm(t, x, exact=True, bias=torch.from_numpy(bias).cuda(), activation=act,
                out_dtype=torch.float16 if f16 else torch.float32)
    v = (want + bias[:, None]).astype(np.float32)  # one fp32 add per element (IEEE RN)
    if act == "relu":
        v = _relu(v)
    if f16:
        assert (y.cpu().numpy().view(np.uint16) == _np_f16_bits(v)).all()
    else:
        assert y.cpu().numpy().tobytes() == v.tobytes()


def test_narrowing_special_values(port):
    """Overflow to inf, subnormal results and the canonical NaN through the epilogue."""
    import torch

    import paper_2309_10285_b200 as tc
    a = np.zeros((128, 64), np.uint16)
    a[0, 0] = np.float16(1.0).view(np.uint16)
    a[1, 0] = np.float16(-1.0).view(np.uint16)
    a[2, 0] = np.float16(1.0).view(np.uint16)
    x = np.zeros((64, 8), np.uint16)
    x[0, :] = np.float16(1.0).view(np.uint16)
    t = tc.encode(torch.from_numpy(a.view(np.int16)).cuda())
    bias = np.zeros(128, np.float32)
    bias[0] = 65519.0 - 1.0   # 1 + 65518 = 65519 -> rounds to 65504
    bias[1] = 1.0 - 65520.0   # -1 + 1 - 65520 -> -inf after RNE (tie to even)
    bias[3] = float("nan")
    bias[4] = 3.0 * 2.0 ** -25  # 0 + 3*2^-25 -> subnormal 2
    for exact in (True, False):
        y = tc.spmm(t, torch.from_numpy(x.view(np.int16)).cuda(), exact=exact, bias=torch.from_numpy(bias).cuda(),
                    out_dtype=torch.float16).cpu().numpy().view(np.uint16)
        assert (y[0] == 0x7BFF).all() and (y[1] == 0xFC00).all() and (y[2] == 0x3C00).all()
        assert (y[3] == 0x7E00).all()
        assert (y[4] == 0x0002).all()
        assert (y[5:] == 0).all()


@pytest.mark.parametrize("split", [1, 3])
@pytest.mark.parametrize("act", [None, "relu", "gelu_tanh"])
@pytest.mark.parametrize("f16", [False, True])
def test_tensor_core_path_within_tolerance(port, split, act, f16):
    import torch

    import paper_2309_10285_b200 as tc
    t, x, want, bound, bias = _case(port, 512, 2048, 32, 0.85, 17)
    y = tc.spmm(t, x, split_k=split, bias=torch.from_numpy(bias).cuda(), activation=act,
                out_dtype=torch.float16 if f16 else torch.float32).cpu().numpy().astype(np.float64)
    v = want.astype(np.float64) + bias[:, None]
    tol = ELEM * bound.astype(np.float64) + np.abs(v) * 2.0 ** -23  # + the fp32 rounding of acc + bias
    if act == "relu":
        v = np.maximum(v, 0)
    elif act == "gelu_tanh":
        v = 0.5 * v * (1 + np.tanh(0.7978845608028654 * (v + 0.044715 * v ** 3)))
        tol = 1.13 * tol + 1e-6 * np.abs(v) + 1e-6  # GELU's slope <= 1.13; tanhf ulps
    if f16:
        tol = tol + np.abs(v) * 2.0 ** -11 + 2.0 ** -25  # half a binary16 ulp
    assert (np.abs(y - v) <= tol).all(), float(np.max(np.abs(y - v) - tol))


def test_non_default_tiles_with_epilogue(port):
    import torch

    import paper_2309_10285_b200 as tc
    a = port.gen_random_sparse(50, 40, 0.6, 3)
    x = port.gen_random_sparse(40, 7, 0.1, 4)
    t = tc.encode(torch.from_numpy(a.view(np.int16)).cuda(), tc.TileConfig(16, 8))
    want = port.spmm(port.encode(a, 16, 8), x)
    bias = np.linspace(-3, 3, 50).astype(np.float32)
    y = tc.spmm(t, torch.from_numpy(x.view(np.int16)).cuda(), bias=torch.from_numpy(bias).cuda(), activation="relu",
                out_dtype=torch.float16)
    assert (y.cpu().numpy().view(np.uint16) == _np_f16_bits(_relu((want + bias[:, None]).astype(np.float32)))).all()
