# column-partitioned layout on one GPU (two ranks, host data plane); full suite
set -x
timeout 900 python -m pytest tests/test_gpu_colshard.py -q -x 2>&1 | tail -30
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6
