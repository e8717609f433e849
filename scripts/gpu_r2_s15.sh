# Gram via DMMA + cp.async: tests, A/B P1/Q1, failing-test details, full suite
set -x
timeout 900 python -m pytest tests/test_gpu_gram.py -q 2>&1 | grep -E "^E |Error|passed|failed" | head -30
timeout 600 python -m pytest "tests/test_gpu_kernels.py::test_column_panels_row_products" -q -x 2>&1 | grep -E "^E |rror" | head -12
for W in P1 Q1; do
  timeout 900 python scripts/ab_kernels.py $W gram
done 2>&1 | grep '^{' | tee gpurun_out/s15_ab.txt
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8
