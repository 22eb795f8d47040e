"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU and
exports exactly the entry points include/tcsl_cuda.h declares; host-side
argument errors map to the reference's Errc classes."""
import ctypes as C
import os
import re

import pytest

import paper_2309_10285_b200 as tc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    with open(os.path.join(ROOT, "include", "tcsl_cuda.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(tcsl_cuda_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(tc.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    tc.build()
    L = tc.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert L.tcsl_cuda_abi_version() == 2
    assert L.tcsl_cuda_status_string(8) == b"location out of range"


def test_host_side_argument_errors():
    L = tc.lib()
    ws = C.c_size_t()
    # TileConfig::validate (matrix.cpp:11-18): multiples of 8, <= 65536 elements
    assert L.tcsl_cuda_encode_workspace(16, 16, 12, 8, C.byref(ws)) == 10
    assert L.tcsl_cuda_encode_workspace(16, 16, 512, 256, C.byref(ws)) == 10
    assert L.tcsl_cuda_encode_workspace(0, 16, 128, 64, C.byref(ws)) == 10
    assert L.tcsl_cuda_encode_workspace(300, 200, 128, 64, C.byref(ws)) == 0 and ws.value > 0
    assert L.tcsl_cuda_spmm_workspace(256, 128, 128, 64, 0, 0, C.byref(ws)) == 10
    # null pointers are rejected before anything touches the device
    assert L.tcsl_cuda_spmm(None, None, 0, 128, 64, 128, 64, None, 8, None, 1, None, 0, None, None) == 10
    assert L.tcsl_cuda_decode(None, None, 0, 0, 64, 128, 64, None, None, None) == 3  # bad_header


def test_auto_split_heuristic_shapes():
    L = tc.lib()
    # tall-K FFN2 9216x36864 (72 row blocks) must split; FFN1 36864x9216 (288) need not
    assert L.tcsl_cuda_spmm_auto_split(9216, 36864, 8) >= 2
    assert L.tcsl_cuda_spmm_auto_split(7168, 7168, 16) >= 2
    assert L.tcsl_cuda_spmm_auto_split(36864, 9216, 8) >= 1


def test_errors_mirror_reference_classes():
    e = tc.TcslError(9, "x")
    assert e.errc == "dimension_mismatch" and e.is_usage()
    assert not tc.TcslError(8).is_usage()
    with pytest.raises(RuntimeError):
        raise tc.TcslError(64, "cuda")
