"""Debug tool: build an experimental variant of the CUDA library for A/B timing.

  python tools/build_variant.py NAME [--rev GITREV] [-DFOO=1 ...]

Compiles csrc/ (spmm_sm100.cu taken from GITREV when given) with the product
flags into paper_2309_10285_b200/_lib/var_NAME.so. Select it at run time with
TCSL_CUDA_LIB=paper_2309_10285_b200/_lib/var_NAME.so."""
import os
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_10285_b200 as tc  # noqa: E402

name, rest = sys.argv[1], sys.argv[2:]
rev, defs = None, []
while rest:
    a = rest.pop(0)
    if a == "--rev":
        rev = rest.pop(0)
    else:
        defs.append(a)
srcs = [os.path.join(tc.CSRC, s) for s in tc.SOURCES]
tmpdir = None
if rev:
    tmpdir = tempfile.mkdtemp(dir=tc.CSRC, prefix=".var_")
    path = os.path.join(tmpdir, "spmm_sm100.cu")
    body = subprocess.run(["git", "show", f"{rev}:paper_2309_10285_b200/csrc/spmm_sm100.cu"], check=True,
                          capture_output=True, text=True).stdout
    open(path, "w").write(body)
    srcs = [path if s.endswith("spmm_sm100.cu") else s for s in srcs]
out = os.path.join(tc.LIB_DIR, f"var_{name}.so")
cmd = ["nvcc", *tc.NVCC_FLAGS, f"-I{tc.CSRC}", *defs, "-o", out, *srcs]
try:
    subprocess.run(cmd, check=True)
finally:
    if tmpdir:
        import shutil
        shutil.rmtree(tmpdir)
print(out)
