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
SOURCES = ["encode.cu", "misc.cu", "spmm_sm100.cu", "capi.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

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
    """Compile csrc/*.cu for sm_100a into _lib/libtcsl_cuda.so (in-tree)."""
    os.makedirs(LIB_DIR, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    newest = max(os.path.getmtime(p) for p in srcs + [os.path.join(CSRC, "sm100_ptx.cuh"),
                                                        os.path.join(CSRC, "tcsl_internal.cuh"),
                                                        os.path.join(HERE, "..", "include", "tcsl_cuda.h")])
    if os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    tmp = LIB_PATH + ".tmp"
    cmd = ["nvcc", *NVCC_FLAGS, "-o", tmp, *srcs]
    subprocess.run(cmd, check=True, capture_output=not verbose)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


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
        "tcsl_cuda_decode": ([vp, vp, u64, u32, u32, i32, i32, vp, vp, vp], i32),
        "tcsl_cuda_validate": ([vp, u64, u32, u32, i32, i32, vp, vp], i32),
        "tcsl_cuda_spmm_workspace": ([u32, u32, i32, i32, i32, i32, C.POINTER(sz)], i32),
        "tcsl_cuda_spmm": ([vp, vp, u64, u32, u32, i32, i32, vp, i32, vp, i32, vp, sz, vp, vp], i32),
        "tcsl_cuda_spmm_auto_split": ([u32, u32, i32], i32),
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
    "tcsl_cuda_validate", "tcsl_cuda_spmm_workspace", "tcsl_cuda_spmm", "tcsl_cuda_spmm_auto_split",
    "tcsl_cuda_splitk_reduce", "tcsl_cuda_spmm_exact_workspace", "tcsl_cuda_spmm_exact",
    "tcsl_cuda_rebase_offsets", "tcsl_cuda_gen_synthetic", "tcsl_cuda_malloc", "tcsl_cuda_free",
    "tcsl_cuda_memcpy_h2d", "tcsl_cuda_memcpy_d2h", "tcsl_cuda_memset", "tcsl_cuda_stream_sync",
    "tcsl_cuda_device_count",
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


def _as_u16(w):
    torch = _torch()
    if w.dtype in (torch.float16, torch.bfloat16, torch.int16):
        w = w.view(torch.int16)
    elif w.dtype == torch.uint16:
        w = w.view(torch.int16)
    else:
        raise TcslError(10, f"expected a 16-bit tensor, got {w.dtype}")
    if not w.is_cuda:
        raise TcslError(10, "tensor must be on the GPU")
    return w.contiguous()


def encode(w, cfg: TileConfig | None = None, reorder: bool = True) -> TcslMatrix:
    """Dense binary16 W[m, k] (GPU) -> TcslMatrix, bit-exact with tcsl::encode."""
    torch = _torch()
    cfg = cfg or TileConfig()
    if w.dim() != 2 or w.shape[0] == 0 or w.shape[1] == 0:
        raise TcslError(10, "cannot encode an empty matrix")
    w = _as_u16(w)
    m, k = w.shape
    L, s = lib(), _stream()
    ws_bytes = C.c_size_t()
    _check(L.tcsl_cuda_encode_workspace(m, k, cfg.m_tb, cfg.k_tb, C.byref(ws_bytes)), "encode")
    T = -(-m // cfg.m_tb) * -(-k // cfg.k_tb)
    off = torch.empty(T + 1, dtype=torch.int32, device=w.device)
    ws = torch.empty(max(ws_bytes.value, 1), dtype=torch.uint8, device=w.device)
    _check(L.tcsl_cuda_encode_count(_ptr(w), m, k, cfg.m_tb, cfg.k_tb, _ptr(off), _ptr(ws), ws_bytes.value, s))
    E = int(off[T].item()) & 0xFFFFFFFF
    ent = torch.empty(E, dtype=torch.int32, device=w.device)
    err = torch.zeros(1, dtype=torch.int32, device=w.device)
    _check(L.tcsl_cuda_encode_emit(_ptr(w), m, k, cfg.m_tb, cfg.k_tb, int(reorder), _ptr(off), _ptr(ent),
                                   _ptr(err), s))
    _check(L.tcsl_cuda_read_error(_ptr(err), s), "encode")
    return TcslMatrix(m, k, cfg, reorder, off, ent)


def decode(t: TcslMatrix):
    """TcslMatrix -> dense binary16 bits [m, k] as int16 (tcsl::decode)."""
    torch = _torch()
    L, s = lib(), _stream()
    out = torch.empty((t.m, t.k), dtype=torch.int16, device=t.offsets.device)
    err = torch.zeros(1, dtype=torch.int32, device=t.offsets.device)
    _check(L.tcsl_cuda_decode(_ptr(t.offsets), _ptr(t.entries), t.n_entries, t.m, t.k, t.cfg.m_tb, t.cfg.k_tb,
                              _ptr(out), _ptr(err), s))
    _check(L.tcsl_cuda_read_error(_ptr(err), s), "decode")
    return out


def validate(t: TcslMatrix) -> None:
    torch = _torch()
    L, s = lib(), _stream()
    err = torch.zeros(1, dtype=torch.int32, device=t.offsets.device)
    if t.offsets.numel() != t.num_tiles + 1:
        raise TcslError(7, "offset table must have num_tiles+1 entries")
    _check(L.tcsl_cuda_validate(_ptr(t.offsets), t.n_entries, t.m, t.k, t.cfg.m_tb, t.cfg.k_tb, _ptr(err), s))
    _check(L.tcsl_cuda_read_error(_ptr(err), s), "validate")


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
         check: bool = True):
    """Y[m, n] fp32 = t @ X[k, n] (X binary16 on the GPU). tcsl::spmm semantics.

    exact=True runs the bit-exact CUDA-core mode (dense_gemm_ref order)."""
    torch = _torch()
    if x.dim() != 2 or x.shape[0] == 0 or x.shape[1] == 0:
        raise TcslError(10, "B must be non-empty")
    if x.shape[0] != t.k:
        raise TcslError(9, f"A has {t.k} columns, B has {x.shape[0]} rows")
    x = _as_u16(x)
    n = x.shape[1]
    L, s = lib(), _stream()
    dev = t.offsets.device
    if out is None:
        out = torch.empty((t.m, n), dtype=torch.float32, device=dev)
    ws = ws or _default_ws
    nb = C.c_size_t()
    if exact:
        _check(L.tcsl_cuda_spmm_exact_workspace(t.m, t.k, C.byref(nb)))
    else:
        _check(L.tcsl_cuda_spmm_workspace(t.m, t.k, t.cfg.m_tb, t.cfg.k_tb, n, split_k, C.byref(nb)))
    buf, err = ws.get(nb.value, dev)
    if check:
        err.zero_()
    fn = L.tcsl_cuda_spmm_exact if exact else L.tcsl_cuda_spmm
    args = [_ptr(t.offsets), _ptr(t.entries), t.n_entries, t.m, t.k, t.cfg.m_tb, t.cfg.k_tb, _ptr(x), n,
            _ptr(out)]
    if not exact:
        args.append(split_k)
    args += [_ptr(buf), buf.numel(), _ptr(err), s]
    _check(fn(*args), "spmm")
    if check:
        _check(L.tcsl_cuda_read_error(_ptr(err), s), "spmm")
    return out


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
    return TcslMatrix(rows, t.k, t.cfg, t.reordered, off, t.entries[lo:hi])


def gen_synthetic(rows: int, cols: int, beta: float, seed: int, device="cuda"):
    """Synthetic random-sparse binary16 bits [rows, cols] (int16) generated on the GPU."""
    torch = _torch()
    w = torch.empty((rows, cols), dtype=torch.int16, device=device)
    _check(lib().tcsl_cuda_gen_synthetic(_ptr(w), rows * cols, float(beta), seed & (2**64 - 1), _stream()))
    return w
