#!/bin/bash
# Builds the TCSL_TRACE debug library (_lib/libtcsl_cuda_trace.so; never used by the product path).
cd "$(dirname "$0")/.." && python - <<'PY'
import os, subprocess, sys
sys.path.insert(0, ".")
import paper_2309_10285_b200 as tc
out = os.path.join(tc.LIB_DIR, "libtcsl_cuda_trace.so")
subprocess.run(["nvcc", *tc.NVCC_FLAGS, "-DTCSL_TRACE", *sys.argv[1:], "-o", out, *[os.path.join(tc.CSRC, f) for f in tc.SOURCES]], check=True)
print(out)
PY
