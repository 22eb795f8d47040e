"""Regenerates tests/golden/* from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists): `python tests/golden/make_golden.py`.
Outputs:
  golden_{a,b,c}.tcsl — the reference's golden artifacts; their FNV-1a hashes
      are pinned in proj/tests/acceptance.cpp:60-64 and re-checked here.
  kats.json — encoder and spmm known answers computed by the reference
      (tcsl::gen_random_sparse -> tcsl::encode -> serialize FNV; tcsl::spmm
      -> FNV of the f32 bytes), used on the GPU box where /root/reference is
      absent.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

GOLDEN = [  # proj/tests/acceptance.cpp:60-64
    ("golden_a.tcsl", 128, 64, 0.3, 11, True, 0xa57f18792a5f0447),
    ("golden_b.tcsl", 256, 128, 0.8, 22, True, 0x2a290613b42e2457),
    ("golden_c.tcsl", 130, 70, 0.5, 33, False, 0xf68ef9afd7dea93a),
]

ENCODE_CASES = [  # (rows, cols, beta, seed, m_tb, k_tb, reorder)
    (128, 64, 0.0, 1, 128, 64, True),
    (128, 64, 1.0, 2, 128, 64, True),
    (300, 150, 0.7, 3, 128, 64, True),
    (300, 150, 0.7, 3, 128, 64, False),
    (1, 1, 0.0, 4, 128, 64, True),
    (700, 33, 0.9, 5, 128, 64, True),
    (33, 20, 0.55, 14, 16, 8, True),
    (333, 257, 0.8, 6, 64, 32, True),
    (513, 130, 0.5, 7, 256, 64, True),
    (100, 1000, 0.95, 8, 8, 512, True),
    (1024, 1024, 0.8, 9, 128, 64, True),
    (257, 4099, 0.9, 10, 128, 64, False),
]

SPMM_CASES = [  # (m, k, n, beta, seed_a, seed_b)
    (128, 64, 8, 0.8, 21, 22),
    (256, 128, 16, 0.8, 23, 24),
    (300, 200, 32, 0.7, 25, 26),
    (1024, 512, 64, 0.9, 27, 28),
    (7168 // 8, 7168 // 4, 16, 0.8, 29, 30),
]


def fnv(b: bytes) -> int:
    return oracle.port().fnv1a(b)


def main() -> None:
    R, P = oracle.ref(), oracle.port()
    for name, r, c, beta, seed, reorder, want in GOLDEN:
        a = R.gen_random_sparse(r, c, beta, seed)
        t, h, _ = R.encode(a, reorder=reorder, with_fnv=True)
        assert h == want, (name, hex(h))
        data = P.serialize(t)
        assert fnv(data) == want
        with open(os.path.join(HERE, name), "wb") as f:
            f.write(data)
    kats = {"encode": [], "spmm": []}
    for (r, c, beta, seed, m_tb, k_tb, reorder) in ENCODE_CASES:
        a = R.gen_random_sparse(r, c, beta, seed)
        t, h, size = R.encode(a, m_tb, k_tb, reorder, with_fnv=True)
        kats["encode"].append(dict(rows=r, cols=c, beta=beta, seed=seed, m_tb=m_tb, k_tb=k_tb,
                                   reorder=reorder, n_entries=int(len(t.entries)), fnv=hex(h),
                                   size=int(size)))
    for (m, k, n, beta, sa, sb) in SPMM_CASES:
        a = R.gen_random_sparse(m, k, beta, sa)
        b = R.gen_random_sparse(k, n, 0.0, sb)
        y = R.spmm(R.encode(a), b, 4)
        kats["spmm"].append(dict(m=m, k=k, n=n, beta=beta, seed_a=sa, seed_b=sb,
                                 y_fnv=hex(fnv(y.tobytes())), y00=float(y[0, 0]),
                                 y_abs_sum=float(np.abs(y).astype(np.float64).sum())))
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(kats, f, indent=1)
    print("wrote golden fixtures")


if __name__ == "__main__":
    main()
