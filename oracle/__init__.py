"""ctypes bindings for the CPU oracles — TEST INFRASTRUCTURE ONLY.

`port` wraps oracle/_build/liboracle.so (the C restatement, tcsl_oracle.c);
`ref` wraps oracle/_ref/libtcsl_ref.so (the unmodified reference sources built
by oracle/Makefile). Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / `--impl reference` legs import this package, as the checker or the
timed CPU baseline; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtcsl_ref.so")

ERRC = ["bad_magic", "bad_version", "bad_header", "bad_dtype", "truncated", "trailing_data",
        "inconsistent_offsets", "location_out_of_range", "dimension_mismatch", "invalid_argument",
        "io_failure"]


class OracleError(RuntimeError):
    def __init__(self, status: int):
        self.status = status
        self.errc = ERRC[status - 1] if 1 <= status <= len(ERRC) else f"status{status}"
        super().__init__(self.errc)


def _check(st: int) -> None:
    if st:
        raise OracleError(st)


def build() -> None:
    """Compile the oracles (the reference one only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


@dataclass
class Tcsl:
    """Host Tiled-CSL matrix (mirrors tcsl::TcslMatrix, tcsl_format.hpp:40-54)."""
    m: int
    k: int
    m_tb: int
    k_tb: int
    reordered: bool
    offsets: np.ndarray  # uint32[T+1]
    entries: np.ndarray  # uint32[E]

    @property
    def tiles_m(self) -> int:
        return -(-self.m // self.m_tb)

    @property
    def tiles_k(self) -> int:
        return -(-self.k // self.k_tb)

    @property
    def num_tiles(self) -> int:
        return self.tiles_m * self.tiles_k


class _OrcTcsl(C.Structure):
    _fields_ = [("m", C.c_uint32), ("k", C.c_uint32), ("m_tb", C.c_int32), ("k_tb", C.c_int32),
                ("reordered", C.c_int32), ("num_tiles", C.c_uint32),
                ("offsets", C.POINTER(C.c_uint32)), ("entries", C.POINTER(C.c_uint32)),
                ("n_entries", C.c_uint64)]


def _p(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class _Port:
    def __init__(self) -> None:
        if not os.path.exists(PORT_SO):
            build()
        self.lib = L = C.CDLL(PORT_SO)
        L.orc_gen_random_sparse.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_void_p]
        L.orc_encode.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                 C.POINTER(C.POINTER(_OrcTcsl))]
        L.orc_tcsl_free.argtypes = [C.POINTER(_OrcTcsl)]
        L.orc_tcsl_view.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                    C.c_void_p, C.c_uint64]
        L.orc_tcsl_view.restype = _OrcTcsl
        for f in ("orc_decode",):
            getattr(L, f).argtypes = [C.POINTER(_OrcTcsl), C.c_void_p]
        L.orc_extract_tile.argtypes = [C.POINTER(_OrcTcsl), C.c_uint32, C.c_void_p]
        L.orc_reg_pressure.argtypes = [C.POINTER(_OrcTcsl), C.c_int, C.POINTER(C.c_int)]
        L.orc_spmm.argtypes = [C.POINTER(_OrcTcsl), C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        L.orc_dense_gemm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                     C.c_int, C.c_void_p]
        L.orc_serialize.argtypes = [C.POINTER(_OrcTcsl), C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
        L.orc_deserialize.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.POINTER(_OrcTcsl))]
        L.orc_fnv1a.argtypes = [C.c_void_p, C.c_size_t]
        L.orc_fnv1a.restype = C.c_uint64
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_prune_magnitude.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_void_p]
        L.orc_f32_from_f16.argtypes = [C.c_uint16]
        L.orc_f32_from_f16.restype = C.c_float
        L.orc_f16_from_f32.argtypes = [C.c_float]
        L.orc_f16_from_f32.restype = C.c_uint16

    # -- helpers -------------------------------------------------------------
    @staticmethod
    def _to_tcsl(p) -> Tcsl:
        t = p.contents
        nt = t.num_tiles
        off = np.ctypeslib.as_array(t.offsets, shape=(nt + 1,)).copy()
        ent = (np.ctypeslib.as_array(t.entries, shape=(t.n_entries,)).copy()
               if t.n_entries else np.zeros(0, np.uint32))
        return Tcsl(t.m, t.k, t.m_tb, t.k_tb, bool(t.reordered), off, ent)

    def _view(self, t: Tcsl):
        off = np.ascontiguousarray(t.offsets, dtype=np.uint32)
        ent = np.ascontiguousarray(t.entries, dtype=np.uint32)
        if ent.size == 0:
            ent = np.zeros(1, np.uint32)
        v = self.lib.orc_tcsl_view(t.m, t.k, t.m_tb, t.k_tb, int(t.reordered), _p(off), _p(ent),
                                   len(t.entries))
        return v, (off, ent)

    # -- API -----------------------------------------------------------------
    def gen_random_sparse(self, rows: int, cols: int, beta: float, seed: int) -> np.ndarray:
        out = np.empty((max(rows, 0), max(cols, 0)), np.uint16)
        _check(self.lib.orc_gen_random_sparse(rows, cols, beta, seed & (2**64 - 1), _p(out)))
        return out

    def encode(self, a: np.ndarray, m_tb: int = 128, k_tb: int = 64, reorder: bool = True) -> Tcsl:
        a = np.ascontiguousarray(a, dtype=np.uint16)
        rows, cols = a.shape if a.ndim == 2 else (0, 0)
        p = C.POINTER(_OrcTcsl)()
        _check(self.lib.orc_encode(_p(a) if a.size else None, rows, cols, m_tb, k_tb, int(reorder),
                                   C.byref(p)))
        try:
            return self._to_tcsl(p)
        finally:
            self.lib.orc_tcsl_free(p)

    def decode(self, t: Tcsl) -> np.ndarray:
        out = np.empty((t.m, t.k), np.uint16)
        v, keep = self._view(t)
        _check(self.lib.orc_decode(C.byref(v), _p(out)))
        return out

    def extract_tile(self, t: Tcsl, tile: int) -> np.ndarray:
        out = np.empty(t.m_tb * t.k_tb, np.uint16)
        v, keep = self._view(t)
        _check(self.lib.orc_extract_tile(C.byref(v), tile, _p(out)))
        return out

    def reg_pressure(self, t: Tcsl, threads: int = 128) -> int:
        v, keep = self._view(t)
        r = C.c_int()
        _check(self.lib.orc_reg_pressure(C.byref(v), threads, C.byref(r)))
        return r.value

    def spmm(self, t: Tcsl, b: np.ndarray, nthreads: int = 1) -> np.ndarray:
        b = np.ascontiguousarray(b, dtype=np.uint16)
        if b.ndim != 2 or b.shape[0] != t.k:
            raise OracleError(9)
        y = np.empty((t.m, b.shape[1]), np.float32)
        v, keep = self._view(t)
        _check(self.lib.orc_spmm(C.byref(v), _p(b), b.shape[1], _p(y), nthreads))
        return y

    def dense_gemm(self, a: np.ndarray, b: np.ndarray, m_tb: int = 128, k_tb: int = 64) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint16)
        b = np.ascontiguousarray(b, dtype=np.uint16)
        if a.shape[1] != b.shape[0]:
            raise OracleError(9)
        y = np.empty((a.shape[0], b.shape[1]), np.float32)
        _check(self.lib.orc_dense_gemm(_p(a), a.shape[0], a.shape[1], _p(b), b.shape[1], m_tb, k_tb,
                                       _p(y)))
        return y

    def serialize(self, t: Tcsl) -> bytes:
        v, keep = self._view(t)
        buf = C.c_void_p()
        size = C.c_size_t()
        _check(self.lib.orc_serialize(C.byref(v), C.byref(buf), C.byref(size)))
        try:
            return C.string_at(buf, size.value)
        finally:
            self.lib.orc_free(buf)

    def deserialize(self, data: bytes) -> Tcsl:
        arr = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
        p = C.POINTER(_OrcTcsl)()
        _check(self.lib.orc_deserialize(_p(arr), len(data), C.byref(p)))
        try:
            return self._to_tcsl(p)
        finally:
            self.lib.orc_tcsl_free(p)

    def fnv1a(self, data: bytes) -> int:
        arr = np.frombuffer(data, np.uint8)
        return self.lib.orc_fnv1a(_p(arr) if len(data) else None, len(data))

    def prune_magnitude(self, a: np.ndarray, beta: float) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint16)
        out = np.empty_like(a)
        _check(self.lib.orc_prune_magnitude(_p(a), a.size, beta, _p(out)))
        return out

    def f32_from_f16(self, b: int) -> float:
        return self.lib.orc_f32_from_f16(b)

    def f16_from_f32(self, v: float) -> int:
        return self.lib.orc_f16_from_f32(v)


class _Ref:
    """The unmodified reference library (oracle/_ref/libtcsl_ref.so)."""

    def __init__(self) -> None:
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.lib = L = C.CDLL(REF_SO)
        L.ref_gen_random_sparse.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_void_p]
        L.ref_encode.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                 C.POINTER(C.c_void_p)]
        L.ref_tcsl_num_tiles.argtypes = [C.c_void_p]
        L.ref_tcsl_num_tiles.restype = C.c_uint32
        L.ref_tcsl_num_entries.argtypes = [C.c_void_p]
        L.ref_tcsl_num_entries.restype = C.c_uint64
        L.ref_tcsl_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_tcsl_free.argtypes = [C.c_void_p]
        L.ref_serialize_fnv.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.ref_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int,
                                 C.c_int, C.c_void_p]
        L.ref_dense_gemm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                     C.c_int, C.c_void_p]
        L.ref_spmm_prepare.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32,
                                       C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_spmm_free.argtypes = [C.c_void_p]
        L.ref_spmm_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]

    def gen_random_sparse(self, rows: int, cols: int, beta: float, seed: int) -> np.ndarray:
        out = np.empty((rows, cols), np.uint16)
        _check(self.lib.ref_gen_random_sparse(rows, cols, beta, seed & (2**64 - 1), _p(out)))
        return out

    def encode(self, a: np.ndarray, m_tb: int = 128, k_tb: int = 64, reorder: bool = True,
               with_fnv: bool = False):
        a = np.ascontiguousarray(a, dtype=np.uint16)
        h = C.c_void_p()
        _check(self.lib.ref_encode(_p(a), a.shape[0], a.shape[1], m_tb, k_tb, int(reorder), C.byref(h)))
        try:
            nt = self.lib.ref_tcsl_num_tiles(h)
            ne = self.lib.ref_tcsl_num_entries(h)
            off = np.empty(nt + 1, np.uint32)
            ent = np.empty(max(ne, 1), np.uint32)
            self.lib.ref_tcsl_copy(h, _p(off), _p(ent))
            t = Tcsl(a.shape[0], a.shape[1], m_tb, k_tb, reorder, off, ent[:ne].copy())
            if with_fnv:
                hv, sz = C.c_uint64(), C.c_uint64()
                _check(self.lib.ref_serialize_fnv(h, C.byref(hv), C.byref(sz)))
                return t, hv.value, sz.value
            return t
        finally:
            self.lib.ref_tcsl_free(h)

    def decode(self, t: Tcsl) -> np.ndarray:
        out = np.empty((t.m, t.k), np.uint16)
        ent = t.entries if t.entries.size else np.zeros(1, np.uint32)
        _check(self.lib.ref_decode(_p(t.offsets), _p(ent), len(t.entries), t.m, t.k, t.m_tb, t.k_tb,
                                   _p(out)))
        return out

    def dense_gemm(self, a: np.ndarray, b: np.ndarray, m_tb: int = 128, k_tb: int = 64) -> np.ndarray:
        y = np.empty((a.shape[0], b.shape[1]), np.float32)
        _check(self.lib.ref_dense_gemm(_p(a), a.shape[0], a.shape[1], _p(b), b.shape[1], m_tb, k_tb,
                                       _p(y)))
        return y

    def spmm_plan(self, t: Tcsl, nshards: int = 1):
        ent = np.ascontiguousarray(t.entries) if t.entries.size else np.zeros(1, np.uint32)
        off = np.ascontiguousarray(t.offsets)
        h = C.c_void_p()
        _check(self.lib.ref_spmm_prepare(_p(off), _p(ent), len(t.entries), t.m, t.k, t.m_tb, t.k_tb,
                                         nshards, C.byref(h)))
        return h

    def spmm_run(self, plan, b: np.ndarray, m: int, y: np.ndarray | None = None) -> np.ndarray:
        b = np.ascontiguousarray(b, dtype=np.uint16)
        if y is None:
            y = np.empty((m, b.shape[1]), np.float32)
        _check(self.lib.ref_spmm_run(plan, _p(b), b.shape[0], b.shape[1], _p(y)))
        return y

    def spmm_free(self, plan) -> None:
        self.lib.ref_spmm_free(plan)

    def spmm(self, t: Tcsl, b: np.ndarray, nthreads: int = 1) -> np.ndarray:
        plan = self.spmm_plan(t, nthreads)
        try:
            return self.spmm_run(plan, b, t.m)
        finally:
            self.spmm_free(plan)


_port = None
_ref = None


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    try:
        ref()
        return True
    except (OSError, FileNotFoundError, subprocess.CalledProcessError):
        return False
