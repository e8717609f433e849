# K1 tight-eps parity vs the reference's solves (scratch/); panel test detail; K1 bench line with parity
set -x
timeout 900 python scripts/parity_k1_tight.py 1e-06 > gpurun_out/parity_K1.log 2>&1; tail -c 3000 gpurun_out/parity_K1.log
timeout 600 python -m pytest "tests/test_gpu_kernels.py::test_column_panels_row_products" -q -x 2>&1 | grep -E "^E |Error|passed|failed" | head -20
