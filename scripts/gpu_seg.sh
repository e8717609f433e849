#!/bin/bash
# Transposed-product iteration: sparse GPU parity tests, then per-kernel times on N1/R1/K1
# (staged u where it fits, and unstaged).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -q -m gpu --timeout 300 -x > gpurun_out/pytest_seg.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_seg.log
for W in ${@:-N1 R1 K1}; do
  echo "$W $(timeout 600 python scripts/profile_n1.py $W 2>&1 | tail -1)"
  [ $W != K1 ] && echo "$W stage=0 $(TRON_B200_STAGE=0 timeout 600 python scripts/profile_n1.py $W 2>&1 | tail -1)"
done
