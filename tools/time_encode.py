"""Debug tool: device time of the GPU encoder (K1) on an OPT-66B weight: two-pass
(count + scan + emit, per-kernel times) and one-pass fused (tcsl_cuda_encode_fused).

  python tools/time_encode.py [M K beta]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_10285_b200 as tc  # noqa: E402

M, K, beta = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (36864, 9216, 0.8)
w = tc.gen_synthetic(M, K, beta, 1)
t = tc.encode(w)
E = t.n_entries
L = tc.lib()
s = torch.cuda.current_stream().cuda_stream
T = t.num_tiles
ws_bytes = C.c_size_t()
L.tcsl_cuda_encode_workspace(M, K, 128, 64, C.byref(ws_bytes))
ws = torch.empty(ws_bytes.value, dtype=torch.uint8, device="cuda")
fws = C.c_size_t()
L.tcsl_cuda_encode_fused_workspace(M, K, 128, 64, C.byref(fws))
fw = torch.empty(fws.value, dtype=torch.uint8, device="cuda")
off = torch.empty(T + 1, dtype=torch.int32, device="cuda")
ent = torch.empty(E, dtype=torch.int32, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


us_c = timed(lambda: L.tcsl_cuda_encode_count(p(w), M, K, 128, 64, p(off), p(ws), ws_bytes.value, s))
us_e = timed(lambda: L.tcsl_cuda_encode_emit(p(w), M, K, 128, 64, 1, p(off), p(ent), p(err), s))
assert torch.equal(ent, t.entries) and torch.equal(off, t.offsets)
ent.zero_()
us_f = timed(lambda: L.tcsl_cuda_encode_fused(p(w), M, K, 128, 64, 1, p(off), p(ent), E, p(fw), fws.value, p(err), s))
assert torch.equal(ent, t.entries) and torch.equal(off, t.offsets)
assert int(err.item()) == 0
dense = 2.0 * M * K
print(f"encode {M}x{K} beta={beta} E={E}: count+scan {us_c:.1f} us ({dense / us_c / 1e3:.0f} GB/s), "
      f"emit {us_e:.1f} us ({(dense + 4 * E) / us_e / 1e3:.0f} GB/s), two-pass {us_c + us_e:.1f} us; "
      f"fused {us_f:.1f} us ({(dense + 4 * E) / us_f / 1e3:.0f} GB/s of 2MK+4E)")
