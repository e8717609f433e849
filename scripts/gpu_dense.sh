#!/bin/bash
# dense-path check: GPU tests touching dense, P1 A/B timings, one ncu capture
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
echo "P1 $(timeout 300 python scripts/profile_n1.py P1 2>&1 | tail -1)"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dense_pass -s 2 -c 2 -o gpurun_out/P1_dense_pass -f python scripts/profile_n1.py P1 > gpurun_out/ncu_P1_dense.log 2>&1
echo ncu rc=$?
