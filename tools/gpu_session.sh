#!/bin/bash
# Session-start check: GPU parity tests, smoke, then an issuer-count A/B on a cell subset.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
VARIANTS=${VARIANTS:-"i1:TCSL_ISSUERS=1 i2:TCSL_ISSUERS=2"} bash tools/gpu_ab2.sh > gpurun_out/ab.txt 2>&1
