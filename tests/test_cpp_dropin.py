"""The C++ drop-in API (include/tcsl/*.hpp -> libtcsl.so -> C-ABI) compiled like a
reference caller: the CPU test builds and links it; the GPU test runs it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2309_10285_b200", "_lib")
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
EXE = os.path.join(LIB, "test_dropin")


def build_exe():
    import paper_2309_10285_b200 as tc
    tc.build()
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2309_10285_b200", "host")], check=True)
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", SRC, "-o", EXE, f"-L{LIB}", "-ltcsl",
                    "-ltcsl_cuda", f"-Wl,-rpath,{LIB}"], check=True)
    return EXE


def test_dropin_builds_and_links():
    exe = build_exe()
    assert os.access(exe, os.X_OK)
    syms = subprocess.run(["nm", "-DC", os.path.join(LIB, "libtcsl.so")], capture_output=True, text=True).stdout
    for name in ("tcsl::encode(", "tcsl::decode(", "tcsl::spmm(", "tcsl::dense_gemm_ref(", "tcsl::serialize_tcsl(",
                 "tcsl::deserialize_tcsl(", "tcsl::extract_tile(", "tcsl::reg_pressure(", "tcsl::gen_random_sparse(",
                 "tcsl::prune_magnitude(", "tcsl::DeviceMatrix::DeviceMatrix(", "tcsl::DeviceMatrix::spmm("):
        assert name in syms, name


def test_dropin_half_conversions_cpu():
    """a8: the drop-in's host binary16 conversions against the reference's
    test_half.cpp cases (exhaustive decode, strided sweep, every midpoint)."""
    build_exe()
    exe = os.path.join(LIB, "test_half_dropin")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", os.path.join(ROOT, "tests", "cpp",
                    "test_half_dropin.cpp"), "-o", exe, f"-L{LIB}", "-ltcsl", "-ltcsl_cuda", f"-Wl,-rpath,{LIB}"],
                   check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_dropin_runs_on_gpu():
    exe = build_exe()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
