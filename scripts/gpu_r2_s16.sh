set -x
timeout 300 python scripts/dbg_panels.py 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_gram.py "tests/test_gpu_kernels.py::test_column_panels_row_products" -q 2>&1 | grep -E "^E |passed|failed" | head -30
