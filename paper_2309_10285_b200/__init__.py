"""B200-native Tiled-CSL (Flash-LLM LSCD) hot path.

Python host mirror of the reference's hot-path interface
(`tcsl::encode`, proj/include/tcsl/tcsl_format.hpp:62; `tcsl::spmm`,
proj/include/tcsl/engine.hpp:18; `tcsl::decode`, tcsl_format.hpp:66) over the
C-ABI in include/tcsl_cuda.h. Tensors live on the GPU (torch is used only for
device memory and streams); every call goes through the in-tree
`_lib/libtcsl_cuda.so`, and there is no CPU fallback: if the library or a
CUDA device is missing the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libtcsl_cuda.so")
if os.environ.get("TCSL_CUDA_LIB"):  # A/B experiments (tools/build_variant.py); still the CUDA library
    LIB_PATH = os.path.abspath(os.environ["TCSL_CUDA_LIB"])
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["encode.cu", "misc.cu", "prune.cu", "spmm_sm100.cu", "capi.cu", "nccl_rows.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-ldl"]

ERRC = ["bad_magic", "bad_version", "bad_header", "bad_dtype", "truncated", "trailing_data",
        "inconsistent_offsets", "location_out_of_range", "dimension_mismatch", "invalid_argument",
        "io_failure"]
STATUS_EXTRA = {64: "cuda_error", 65: "unsupported", 66: "workspace"}


class TcslError(RuntimeError):
    """Mirrors tcsl::Error (proj/include/tcsl/errors.hpp:26-43)."""

    def __init__(self, status: int, detail: str = ""):
        self.status = status
        if 1 <= status <= len(ERRC):
            self.errc = ERRC[status - 1]
        else:
            self.errc = STATUS_EXTRA.get(status, f"status{status}")
        super().__init__(f"{self.errc}{': ' + detail if detail else ''}")

    def is_usage(self) -> bool:  # errors.hpp:35-37
        return self.errc in ("dimension_mismatch", "invalid_argument")


def build(verbose: bool = False) -> str:
    """Compile csrc/*.cu for sm_100a into _lib/libtcsl_cuda.so (in-tree). Each source
    is compiled to its own object (in parallel, only when it or a header changed),
    then linked."""
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(os.path.join(LIB_DIR, "obj"), exist_ok=True)
    headers = [os.path.join(CSRC, "sm100_ptx.cuh"), os.path.join(CSRC, "tcsl_internal.cuh"),
               os.path.join(HERE, "..", "include", "tcsl_cuda.h")]
    hdr_time = max(os.path.getmtime(h) for h in headers)
    objs, todo = [], []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        obj = os.path.join(LIB_DIR, "obj", src.replace(".cu", ".o"))
        objs.append(obj)
        if not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(sp), hdr_time):
            todo.append((sp, obj))
    flags = [f for f in NVCC_FLAGS if f not in ("-shared", "-ldl")]

    def compile_one(job):
        sp, obj = job
        subprocess.run(["nvcc", *flags, "-c", "-o", obj + ".tmp", sp], check=True, capture_output=not verbose)
        os.replace(obj + ".tmp", obj)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(compile_one, todo))
    if todo or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB_PATH + ".tmp"
        subprocess.run(["nvcc", *NVCC_FLAGS, "-o", tmp, *objs], check=True, capture_output=not verbose)
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


class Header(C.Structure):
    """tcsl_cuda_header (include/tcsl_cuda.h)."""
    _fields_ = [("m", C.c_uint32), ("k", C.c_uint32), ("m_tb", C.c_uint32), ("k_tb", C.c_uint32),
                ("num_tiles", C.c_uint32), ("reordered", C.c_uint32), ("n_entries", C.c_uint64)]


# include/tcsl_cuda.h constants
CHECK_SPMM, CHECK_DECODE, CHECK_INGEST = 0, 1, 2
FLAG_DUPLICATE_LOCATIONS, FLAG_PARTIAL_GROUPS, FLAG_FRINGE_PAYLOAD, FLAG_LOCATION_RANGE = 1, 2, 4, 8
ACTIVATIONS = {None: 0, "none": 0, "relu": 1, "gelu_tanh": 2}

_lib = None


def lib() -> C.CDLL:
    """The C-ABI library. Raises if it has not been built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (nvcc, sm_100a)")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32, sz = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_size_t
    sig = {
        "tcsl_cuda_abi_version": ([], i32),
        "tcsl_cuda_status_string": ([i32], C.c_char_p),
        "tcsl_cuda_last_cuda_error": ([], C.c_char_p),
        "tcsl_cuda_read_error": ([vp, vp], i32),
        "tcsl_cuda_encode_workspace": ([u32, u32, i32, i32, C.POINTER(sz)], i32),
        "tcsl_cuda_encode_count": ([vp, u32, u32, i32, i32, vp, vp, sz, vp], i32),
        "tcsl_cuda_encode_emit": ([vp, u32, u32, i32, i32, i32, vp, vp, vp, vp], i32),
        "tcsl_cuda_encode_fused_workspace": ([u32, u32, i32, i32, C.POINTER(sz)], i32),
        "tcsl_cuda_encode_fused": ([vp, u32, u32, i32, i32, i32, vp, vp, u64, vp, sz, vp, vp], i32),
        "tcsl_cuda_decode": ([vp, vp, u64, u32, u32, i32, i32, vp, vp, vp], i32),
        "tcsl_cuda_validate": ([vp, u64, u32, u32, i32, i32, vp, vp], i32),
        "tcsl_cuda_spmm_workspace": ([u32, u32, i32, i32, i32, i32, C.POINTER(sz)], i32),
        "tcsl_cuda_spmm": ([vp, vp, u64, u32, u32, i32, i32, vp, i32, vp, i32, vp, sz, vp, vp], i32),
        "tcsl_cuda_spmm_auto_split": ([u32, u32, i32], i32),
        "tcsl_cuda_spmm_estimate": ([u32, u32, i32, u64, i32, C.c_double, C.POINTER(Estimate)], i32),
        "tcsl_cuda_splitk_reduce": ([vp, i32, sz, vp, vp], i32),
        "tcsl_cuda_spmm_exact_workspace": ([u32, u32, C.POINTER(sz)], i32),
        "tcsl_cuda_spmm_exact": ([vp, vp, u64, u32, u32, i32, i32, vp, i32, vp, vp, sz, vp, vp], i32),
        "tcsl_cuda_rebase_offsets": ([vp, u32, u32, vp, vp], i32),
        "tcsl_cuda_gen_synthetic": ([vp, u64, C.c_double, u64, vp], i32),
        "tcsl_cuda_malloc": ([C.POINTER(vp), sz], i32),
        "tcsl_cuda_free": ([vp], i32),
        "tcsl_cuda_memcpy_h2d": ([vp, vp, sz, vp], i32),
        "tcsl_cuda_memcpy_d2h": ([vp, vp, sz, vp], i32),
        "tcsl_cuda_memset": ([vp, i32, sz, vp], i32),
        "tcsl_cuda_stream_sync": ([vp], i32),
        "tcsl_cuda_device_count": ([C.POINTER(i32)], i32),
        "tcsl_cuda_validate_entries": ([vp, vp, u64, u32, u32, i32, i32, i32, vp, vp, vp], i32),
        "tcsl_cuda_parse_header": ([vp, sz, C.POINTER(Header)], i32),
        "tcsl_cuda_ingest": ([vp, sz, C.POINTER(Header), vp, vp, vp, sz, vp, vp, vp], i32),
        "tcsl_cuda_spmm_ex_workspace": ([u32, u32, i32, i32, i32, i32, i32, C.POINTER(sz)], i32),
        "tcsl_cuda_spmm_ex": ([vp, vp, u64, u32, u32, i32, i32, vp, i32, vp, i32, vp, i32, i32, i32, vp, sz, vp,
                               vp], i32),
        "tcsl_cuda_spmm_push": ([vp, vp, u64, u32, u32, i32, i32, vp, i32, vp, i32, i32, vp, i32, i32, i32, vp, sz,
                                 vp, vp], i32),
        "tcsl_cuda_prune_workspace": ([u64, C.POINTER(sz)], i32),
        "tcsl_cuda_prune_magnitude": ([vp, u64, C.c_double, vp, vp, sz, vp], i32),
        "tcsl_cuda_nccl_available": ([], i32),
        "tcsl_cuda_nccl_unique_id": ([vp], i32),
        "tcsl_cuda_nccl_comm_init": ([C.POINTER(vp), i32, vp, i32], i32),
        "tcsl_cuda_nccl_comm_destroy": ([vp], i32),
        "tcsl_cuda_allgather_rows": ([vp, vp, sz, i32, i32, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


EXPORTED_SYMBOLS = [
    "tcsl_cuda_abi_version", "tcsl_cuda_status_string", "tcsl_cuda_last_cuda_error", "tcsl_cuda_read_error",
    "tcsl_cuda_encode_workspace", "tcsl_cuda_encode_count", "tcsl_cuda_encode_emit", "tcsl_cuda_decode",
    "tcsl_cuda_encode_fused_workspace", "tcsl_cuda_encode_fused", "tcsl_cuda_validate", "tcsl_cuda_spmm_workspace",
    "tcsl_cuda_spmm", "tcsl_cuda_spmm_auto_split", "tcsl_cuda_spmm_estimate",
    "tcsl_cuda_splitk_reduce", "tcsl_cuda_spmm_exact_workspace", "tcsl_cuda_spmm_exact",
    "tcsl_cuda_rebase_offsets", "tcsl_cuda_gen_synthetic", "tcsl_cuda_malloc", "tcsl_cuda_free",
    "tcsl_cuda_memcpy_h2d", "tcsl_cuda_memcpy_d2h", "tcsl_cuda_memset", "tcsl_cuda_stream_sync",
    "tcsl_cuda_device_count", "tcsl_cuda_validate_entries", "tcsl_cuda_parse_header", "tcsl_cuda_ingest",
    "tcsl_cuda_spmm_ex_workspace", "tcsl_cuda_spmm_ex", "tcsl_cuda_spmm_push", "tcsl_cuda_prune_workspace",
    "tcsl_cuda_prune_magnitude",
    "tcsl_cuda_nccl_available", "tcsl_cuda_nccl_unique_id", "tcsl_cuda_nccl_comm_init",
    "tcsl_cuda_nccl_comm_destroy", "tcsl_cuda_allgather_rows",
]


def _check(st: int, what: str = "") -> None:
    if st:
        detail = what
        if st == 64:
            detail = (what + " " + lib().tcsl_cuda_last_cuda_error().decode()).strip()
        raise TcslError(st, detail)


# --------------------------------------------------------------------------- torch side
def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2309_10285_b200 needs a CUDA device (sm_100a); there is no CPU path")
    return torch


def _stream():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() else C.c_void_p(0)


@dataclass
class TileConfig:
    """proj/include/tcsl/matrix.hpp:22-29."""
    m_tb: int = 128
    k_tb: int = 64
    threads_per_block: int = 128


@dataclass
class TcslMatrix:
    """Device-resident Tiled-CSL matrix (tcsl::TcslMatrix, tcsl_format.hpp:40-54).

    offsets: int32 tensor [T+1] holding uint32 bits; entries: int32 tensor [E]
    holding the packed uint32 words (value << 16 | x*k_tb + y)."""
    m: int
    k: int
    cfg: TileConfig
    reordered: bool
    offsets: object
    entries: object
    # True when every tile span is whole 32-entry groups and no location repeats
    # inside a tile (what encode() emits): the tensor-core path's preconditions.
    # None = not known yet: spmm() validates on the device once and caches it.
    tc_ready: bool | None = None

    @property
    def tiles_m(self) -> int:
        return -(-self.m // self.cfg.m_tb)

    @property
    def tiles_k(self) -> int:
        return -(-self.k // self.cfg.k_tb)

    @property
    def num_tiles(self) -> int:
        return self.tiles_m * self.tiles_k

    @property
    def n_entries(self) -> int:
        return int(self.entries.numel())

    def to_host(self):
        """(offsets uint32 ndarray, entries uint32 ndarray)."""
        import numpy as np
        off = self.offsets.cpu().numpy().view(np.uint32)
        ent = self.entries.cpu().numpy().view(np.uint32)
        return off, ent

    @staticmethod
    def from_host(m, k, offsets, entries, cfg: TileConfig | None = None, reordered=True, device="cuda"):
        import numpy as np
        torch = _torch()
        off = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.uint32).view(np.int32)).to(device)
        ent = torch.from_numpy(np.ascontiguousarray(entries, dtype=np.uint32).view(np.int32)).to(device)
        return TcslMatrix(int(m), int(k), cfg or TileConfig(), bool(reordered), off, ent)

    def shares_storage(self, other: "TcslMatrix") -> bool:
        return self.offsets.data_ptr() == other.offsets.data_ptr() and self.entries.data_ptr() == other.entries.data_ptr()


def _as_u16(w):
    """binary16 operands only (the reference API is Eigen::half): float16 values, or
    int16/uint16 tensors holding binary16 bit patterns. bfloat16 is rejected (its
    bits would be misread as binary16)."""
    torch = _torch()
    if w.dtype in (torch.float16, torch.int16, torch.uint16):
        w = w.view(torch.int16)
    else:
        raise TcslError(10, f"expected binary16 (float16, or int16/uint16 bit patterns), got {w.dtype}")
    if not w.is_cuda:
        raise TcslError(10, "tensor must be on the GPU")
    return w.contiguous()


def encode(w, cfg: TileConfig | None = None, reorder: bool = True, capacity: int | None = None) -> TcslMatrix:
    """Dense binary16 W[m, k] (GPU) -> TcslMatrix, bit-exact with tcsl::encode.

    Default: two passes (count + scan, then emit into an exactly sized buffer).
    capacity=C (entries): one pass that reads W once (tcsl_cuda_encode_fused,
    TileConfig {128, 64} with the reorder) into a C-entry buffer; the result is
    a view of its first E entries. If E > C the emit pass runs into an exactly
    sized buffer with the offsets the fused pass computed."""
    torch = _torch()
    cfg = cfg or TileConfig()
    if w.dim() != 2 or w.shape[0] == 0 or w.shape[1] == 0:
        raise TcslError(10, "cannot encode an empty matrix")
    w = _as_u16(w)
    m, k = w.shape
    L, s = lib(), _stream()
    T = -(-m // cfg.m_tb) * -(-k // cfg.k_tb)
    off = torch.empty(T + 1, dtype=torch.int32, device=w.device)
    err = torch.zeros(1, dtype=torch.int32, device=w.device)
    if capacity is not None and reorder and (cfg.m_tb, cfg.k_tb) == (128, 64):
        ws_bytes = C.c_size_t()
        _check(L.tcsl_cuda_encode_fused_workspace(m, k, cfg.m_tb, cfg.k_tb, C.byref(ws_bytes)), "encode")
        ws = torch.empty(max(ws_bytes.value, 1), dtype=torch.uint8, device=w.device)
        buf = torch.empty(max(int(capacity), 4), dtype=torch.int32, device=w.device)
        _check(L.tcsl_cuda_encode_fused(_ptr(w), m, k, cfg.m_tb, cfg.k_tb, 1, _ptr(off), _ptr(buf), int(capacity),
                                        _ptr(ws), ws_bytes.value, _ptr(err), s), "encode")
        E = int(off[T].item()) & 0xFFFFFFFF
        if E <= capacity:
            _check(L.tcsl_cuda_read_error(_ptr(err), s), "encode")
            return TcslMatrix(m, k, cfg, reorder, off, buf[:E], tc_ready=True)
    else:
        ws_bytes = C.c_size_t()
        _check(L.tcsl_cuda_encode_workspace(m, k, cfg.m_tb, cfg.k_tb, C.byref(ws_bytes)), "encode")
        ws = torch.empty(max(ws_bytes.value, 1), dtype=torch.uint8, device=w.device)
        _check(L.tcsl_cuda_encode_count(_ptr(w), m, k, cfg.m_tb, cfg.k_tb, _ptr(off), _ptr(ws), ws_bytes.value, s))
        E = int(off[T].item()) & 0xFFFFFFFF
    ent = torch.empty(E, dtype=torch.int32, device=w.device)
    _check(L.tcsl_cuda_encode_emit(_ptr(w), m, k, cfg.m_tb, cfg.k_tb, int(reorder), _ptr(off), _ptr(ent),
                                   _ptr(err), s))
    _check(L.tcsl_cuda_read_error(_ptr(err), s), "encode")
    return TcslMatrix(m, k, cfg, reorder, off, ent, tc_ready=True)


def decode(t: TcslMatrix):
    """TcslMatrix -> dense binary16 bits [m, k] as int16 (tcsl::decode)."""
    torch = _torch()
    if t.offsets.numel() != t.num_tiles + 1:
        raise TcslError(7, "offset table must have num_tiles+1 entries")
    L, s = lib(), _stream()
    out = torch.empty((t.m, t.k), dtype=torch.int16, device=t.offsets.device)
    err = torch.zeros(1, dtype=torch.int32, device=t.offsets.device)
    _check(L.tcsl_cuda_decode(_ptr(t.offsets), _ptr(t.entries), t.n_entries, t.m, t.k, t.cfg.m_tb, t.cfg.k_tb,
                              _ptr(out), _ptr(err), s))
    _check(L.tcsl_cuda_read_error(_ptr(err), s), "decode")
    return out


def validate(t: TcslMatrix) -> None:
    """check_offsets (proj/src/tcsl_format.cpp:19-32) on the device."""
    torch = _torch()
    L, s = lib(), _stream()
    err = torch.zeros(1, dtype=torch.int32, device=t.offsets.device)
    if t.offsets.numel() != t.num_tiles + 1:
        raise TcslError(7, "offset table must have num_tiles+1 entries")
    _check(L.tcsl_cuda_validate(_ptr(t.offsets), t.n_entries, t.m, t.k, t.cfg.m_tb, t.cfg.k_tb, _ptr(err), s))
    _check(L.tcsl_cuda_read_error(_ptr(err), s), "validate")


def check_entries(t: TcslMatrix, mode: int = CHECK_DECODE) -> int:
    """Whole-matrix validation on the device (tcsl_cuda_validate_entries): raises
    the reference's error class for `mode`'s checks and returns the TCSL_FLAG_* bits."""
    torch = _torch()
    L, s = lib(), _stream()
    if t.offsets.numel() != t.num_tiles + 1:
        raise TcslError(7, "offset table must have num_tiles+1 entries")
    buf = torch.zeros(2, dtype=torch.int32, device=t.offsets.device)  # [error, flags]
    _check(L.tcsl_cuda_validate_entries(_ptr(t.offsets), _ptr(t.entries), t.n_entries, t.m, t.k, t.cfg.m_tb,
                                        t.cfg.k_tb, mode, C.c_void_p(buf.data_ptr() + 4), _ptr(buf), s))
    _check(L.tcsl_cuda_read_error(_ptr(buf), s), "validate")
    return int(buf[1].item())


def _tc_ready(t: TcslMatrix) -> bool:
    """The tensor-core path's preconditions (include/tcsl_cuda.h), checked once per matrix."""
    if t.tc_ready is None:
        flags = check_entries(t, CHECK_SPMM)
        t.tc_ready = not (flags & (FLAG_DUPLICATE_LOCATIONS | FLAG_PARTIAL_GROUPS)) and t.entries.data_ptr() % 16 == 0
    return t.tc_ready


class SpmmWorkspace:
    """Reusable device workspace + error word for repeated spmm calls."""

    def __init__(self):
        self.buf = None
        self.err = None

    def get(self, nbytes: int, device):
        torch = _torch()
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        if self.err is None or self.err.device != device:
            self.err = torch.zeros(1, dtype=torch.int32, device=device)
        return self.buf, self.err


_default_ws = SpmmWorkspace()


def spmm(t: TcslMatrix, x, split_k: int = 0, exact: bool = False, out=None, ws: SpmmWorkspace | None = None,
         check: bool = True, bias=None, activation: str | None = None, out_dtype=None):
    """Y[m, n] = t @ X[k, n] (X binary16 on the GPU). tcsl::spmm semantics.

    exact=True runs the bit-exact CUDA-core mode (dense_gemm_ref order). Inputs
    outside the tensor-core path's preconditions (repeated locations inside a
    tile, spans that are not whole 32-entry groups — both legal for the
    reference's spmm, engine.cpp:8-25) also take the exact path. Optional fused
    epilogue: Y = activation(W X + bias) (bias: fp32 [m]; activation None /
    "relu" / "gelu_tanh"), returned as float32 or, with out_dtype=torch.float16,
    narrowed like f16_from_f32 (proj/src/half.cpp:10-40)."""
    torch = _torch()
    if x.dim() != 2 or x.shape[0] == 0 or x.shape[1] == 0:
        raise TcslError(10, "B must be non-empty")
    if x.shape[0] != t.k:
        raise TcslError(9, f"A has {t.k} columns, B has {x.shape[0]} rows")
    x = _as_u16(x)
    n = x.shape[1]
    dev = t.offsets.device
    if x.device != dev or t.entries.device != dev:
        raise TcslError(10, "A and B must be on the same device")
    if t.offsets.numel() != t.num_tiles + 1:
        raise TcslError(7, "offset table must have num_tiles+1 entries")
    if activation not in ACTIVATIONS:
        raise TcslError(10, f"unknown activation {activation!r}")
    act = ACTIVATIONS[activation]
    out_dtype = out_dtype or (out.dtype if out is not None else torch.float32)
    if out_dtype not in (torch.float32, torch.float16):
        raise TcslError(10, f"output dtype must be float32 or float16, got {out_dtype}")
    f16 = out_dtype == torch.float16
    if out is None:
        out = torch.empty((t.m, n), dtype=out_dtype, device=dev)
    elif (tuple(out.shape) != (t.m, n) or out.dtype != out_dtype or not out.is_contiguous()
          or out.device != dev):
        raise TcslError(10, f"out must be a contiguous {out_dtype} tensor of shape ({t.m}, {n}) on {dev}")
    if bias is not None:
        if bias.dtype != torch.float32 or bias.numel() != t.m or bias.device != dev or not bias.is_contiguous():
            raise TcslError(10, f"bias must be a contiguous float32 tensor of {t.m} elements on {dev}")
    if not exact and t.cfg.m_tb == 128 and t.cfg.k_tb == 64 and not _tc_ready(t):
        exact = True
    L, s = lib(), _stream()
    ws = ws or _default_ws
    nb = C.c_size_t()
    _check(L.tcsl_cuda_spmm_ex_workspace(t.m, t.k, t.cfg.m_tb, t.cfg.k_tb, n, split_k, int(exact), C.byref(nb)))
    buf, err = ws.get(nb.value, dev)
    if check:
        err.zero_()
    _check(L.tcsl_cuda_spmm_ex(_ptr(t.offsets), _ptr(t.entries), t.n_entries, t.m, t.k, t.cfg.m_tb, t.cfg.k_tb,
                               _ptr(x), n, _ptr(out), int(f16), _ptr(bias), act, split_k, int(exact), _ptr(buf),
                               buf.numel(), _ptr(err), s), "spmm")
    if check:
        _check(L.tcsl_cuda_read_error(_ptr(err), s), "spmm")
    return out


def spmm_push(t: TcslMatrix, x, peer_ptrs, split_k: int = 0, exact: bool = False, ws: SpmmWorkspace | None = None,
              check: bool = True, bias=None, activation: str | None = None, out_dtype=None) -> None:
    """Row-shard SpMM with the all-gather fused into the epilogue (tcsl_cuda_spmm_push):
    Y = activation(t @ X + bias) is stored into every destination of `peer_ptrs` (an int64
    device tensor of device addresses — each rank's full-Y buffer offset to this shard's
    first row, e.g. symmetric-memory peer buffers) instead of a local output. The
    caller's cross-rank barrier then makes the rows visible (sharding.RowShardedSpmm)."""
    torch = _torch()
    if x.dim() != 2 or x.shape[0] != t.k or x.shape[1] == 0:
        raise TcslError(9, f"A has {t.k} columns, B has {x.shape[0] if x.dim() == 2 else '?'} rows")
    x = _as_u16(x)
    n = x.shape[1]
    dev = t.offsets.device
    if x.device != dev or peer_ptrs.device != dev or peer_ptrs.dtype != torch.int64 or peer_ptrs.dim() != 1:
        raise TcslError(10, "X and peer_ptrs (int64 addresses) must be on the matrix's device")
    if t.offsets.numel() != t.num_tiles + 1:
        raise TcslError(7, "offset table must have num_tiles+1 entries")
    if activation not in ACTIVATIONS:
        raise TcslError(10, f"unknown activation {activation!r}")
    out_dtype = out_dtype or torch.float32
    if out_dtype not in (torch.float32, torch.float16):
        raise TcslError(10, f"output dtype must be float32 or float16, got {out_dtype}")
    if bias is not None and (bias.dtype != torch.float32 or bias.numel() != t.m or bias.device != dev):
        raise TcslError(10, f"bias must be a float32 tensor of {t.m} elements on {dev}")
    if not exact and t.cfg.m_tb == 128 and t.cfg.k_tb == 64 and not _tc_ready(t):
        exact = True
    L, s = lib(), _stream()
    ws = ws or _default_ws
    nb = C.c_size_t()
    _check(L.tcsl_cuda_spmm_ex_workspace(t.m, t.k, t.cfg.m_tb, t.cfg.k_tb, n, split_k, int(exact), C.byref(nb)))
    buf, err = ws.get(nb.value, dev)
    if check:
        err.zero_()
    _check(L.tcsl_cuda_spmm_push(_ptr(t.offsets), _ptr(t.entries), t.n_entries, t.m, t.k, t.cfg.m_tb, t.cfg.k_tb,
                                 _ptr(x), n, _ptr(peer_ptrs), peer_ptrs.numel(), int(out_dtype == torch.float16),
                                 _ptr(bias), ACTIVATIONS[activation], split_k, int(exact), _ptr(buf), buf.numel(),
                                 _ptr(err), s), "spmm")
    if check:
        _check(L.tcsl_cuda_read_error(_ptr(err), s), "spmm")


class Estimate(C.Structure):
    _fields_ = [("us", C.c_double), ("hbm_us", C.c_double), ("tensor_us", C.c_double), ("smem_us", C.c_double),
                ("chain_us", C.c_double), ("fixed_us", C.c_double), ("split", C.c_int), ("bound", C.c_int)]


BOUNDS = ("hbm", "tensor", "smem", "chain")


def estimate(m: int, k: int, n: int, n_entries: int, split_k: int = 0, hbm_gbs: float = 0.0) -> dict:
    """A-priori B200 time of spmm (tcsl_cuda_spmm_estimate; the B200 counterpart of
    the reference's estimate_time, proj/src/pipeline.cpp:214-273). Host only."""
    e = Estimate()
    _check(lib().tcsl_cuda_spmm_estimate(m, k, n, n_entries, split_k, float(hbm_gbs), C.byref(e)), "estimate")
    return {"us": e.us, "hbm_us": e.hbm_us, "tensor_us": e.tensor_us, "smem_us": e.smem_us,
            "chain_us": e.chain_us, "fixed_us": e.fixed_us, "split": e.split, "bound": BOUNDS[e.bound]}


def auto_split(m: int, k: int, n: int) -> int:
    return lib().tcsl_cuda_spmm_auto_split(m, k, n)


def shard_rows(t: TcslMatrix, tr0: int, tr1: int) -> TcslMatrix:
    """Row shard [tr0*m_tb, min(m, tr1*m_tb)) as a view: rebased offsets + entry slice.

    Bit-identical to encoding that row block."""
    torch = _torch()
    tk = t.tiles_k
    t0, t1 = tr0 * tk, tr1 * tk
    off = torch.empty(t1 - t0 + 1, dtype=torch.int32, device=t.offsets.device)
    _check(lib().tcsl_cuda_rebase_offsets(_ptr(t.offsets), t0, t1, _ptr(off), _stream()))
    lo = int(t.offsets[t0].item()) & 0xFFFFFFFF
    hi = int(t.offsets[t1].item()) & 0xFFFFFFFF
    rows = min(t.m, tr1 * t.cfg.m_tb) - tr0 * t.cfg.m_tb
    return TcslMatrix(rows, t.k, t.cfg, t.reordered, off, t.entries[lo:hi], tc_ready=t.tc_ready)


def gen_synthetic(rows: int, cols: int, beta: float, seed: int, device="cuda"):
    """Synthetic random-sparse binary16 bits [rows, cols] (int16) generated on the GPU."""
    torch = _torch()
    w = torch.empty((rows, cols), dtype=torch.int16, device=device)
    _check(lib().tcsl_cuda_gen_synthetic(_ptr(w), rows * cols, float(beta), seed & (2**64 - 1), _stream()))
    return w


# ------------------------------------------------------------------ TCSL container ingest
def load_tcsl(path_or_bytes, device="cuda") -> TcslMatrix:
    """deserialize_tcsl (proj/src/tcsl_format.cpp:180-222) straight to the device:
    host header checks, pinned-staging upload, structural validation on the GPU
    (no host check_offsets pass). The matrix's tensor-core readiness (no repeated
    locations, whole groups) comes from the same device pass."""
    import numpy as np
    torch = _torch()
    if isinstance(path_or_bytes, (bytes, bytearray, memoryview)):
        data = np.frombuffer(path_or_bytes, dtype=np.uint8)
    else:
        data = np.fromfile(path_or_bytes, dtype=np.uint8)
    L, s = lib(), _stream()
    h = Header()
    _check(L.tcsl_cuda_parse_header(C.c_void_p(data.ctypes.data) if data.size else None, data.size, C.byref(h)),
           "deserialize")
    dev = torch.device(device)
    off = torch.empty(h.num_tiles + 1, dtype=torch.int32, device=dev)
    ent = torch.empty(max(h.n_entries, 1), dtype=torch.int32, device=dev)[: h.n_entries]
    staging = torch.empty(8 << 20, dtype=torch.uint8).pin_memory()
    buf = torch.zeros(2, dtype=torch.int32, device=dev)  # [error, flags]
    _check(L.tcsl_cuda_ingest(C.c_void_p(data.ctypes.data), data.size, C.byref(h), _ptr(off),
                              C.c_void_p(ent.data_ptr()), C.c_void_p(staging.data_ptr()), staging.numel(),
                              C.c_void_p(buf.data_ptr() + 4), _ptr(buf), s), "deserialize")
    _check(L.tcsl_cuda_read_error(_ptr(buf), s), "deserialize")
    flags = int(buf[1].item())
    cfg = TileConfig(int(h.m_tb), int(h.k_tb))
    t = TcslMatrix(int(h.m), int(h.k), cfg, bool(h.reordered), off, ent)
    t.tc_ready = not (flags & (FLAG_DUPLICATE_LOCATIONS | FLAG_PARTIAL_GROUPS | FLAG_LOCATION_RANGE))
    t.ingest_flags = flags
    return t


def serialize_tcsl(t: TcslMatrix) -> bytes:
    """serialize_tcsl (proj/src/tcsl_format.cpp:157-178) of a device matrix: the
    reference's byte layout (28-byte header, offsets, entries)."""
    import struct
    validate(t)
    off, ent = t.to_host()
    head = b"TCSL" + struct.pack("<HHIIIII", 1, 1 if t.reordered else 0, t.m, t.k, t.cfg.m_tb, t.cfg.k_tb,
                                 t.num_tiles)
    return head + off.tobytes() + ent.tobytes()


# ------------------------------------------------------------------ pruning
def prune_magnitude(w, beta: float, out=None):
    """prune_magnitude (proj/src/matrix.cpp:69-100) on the GPU: the floor(beta*n)
    smallest-magnitude elements become +0.0 (ties: larger index first). Returns
    binary16 bits as int16 (out may alias w)."""
    torch = _torch()
    w = _as_u16(w)
    n = w.numel()
    if out is None:
        out = torch.empty_like(w)
    L, s = lib(), _stream()
    nb = C.c_size_t()
    _check(L.tcsl_cuda_prune_workspace(n, C.byref(nb)))
    ws = torch.empty(max(nb.value, 256), dtype=torch.uint8, device=w.device)
    _check(L.tcsl_cuda_prune_magnitude(_ptr(w), n, float(beta), _ptr(out), _ptr(ws), ws.numel(), s), "prune")
    return out


# ------------------------------------------------------------------ multi-GPU (NCCL via the C-ABI)
class RowComm:
    """An NCCL communicator owned by the C-ABI (tcsl_cuda_nccl_comm_init) for the
    row-sharded all-gather of Y. The unique id travels over the
    caller's torch.distributed group (any backend)."""

    def __init__(self, rank: int, world: int, group=None):
        import torch.distributed as dist
        torch = _torch()
        L = lib()
        if not L.tcsl_cuda_nccl_available():
            raise TcslError(65, "libnccl.so.2 not found")
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            _check(L.tcsl_cuda_nccl_unique_id(C.c_void_p(uid.data_ptr())), "nccl id")
        if world > 1:
            backend = dist.get_backend(group)
            t = uid.cuda() if backend == "nccl" else uid
            dist.broadcast(t, 0, group=group)
            uid = t.cpu()
        self.comm = C.c_void_p()
        _check(L.tcsl_cuda_nccl_comm_init(C.byref(self.comm), world, C.c_void_p(uid.data_ptr()), rank), "nccl init")
        self.rank, self.world = rank, world

    def allgather_rows(self, y_local, y_full):
        """y_full[world * rows, n] = concat over ranks of y_local[rows, n] (fp32 or fp16)."""
        torch = _torch()
        f16 = y_local.dtype == torch.float16
        rows, n = y_local.shape
        _check(lib().tcsl_cuda_allgather_rows(_ptr(y_local), _ptr(y_full), rows, n, int(f16), self.comm, _stream()),
               "allgather")
        return y_full

    def close(self):
        if self.comm:
            lib().tcsl_cuda_nccl_comm_destroy(self.comm)
            self.comm = C.c_void_p()
