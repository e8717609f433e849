# dense Gram mode: tests, A/B on P1/Q1, full suite
set -x
timeout 900 python -m pytest tests/test_gpu_gram.py -q -x 2>&1 | tail -25
for W in P1 Q1; do
  timeout 900 python scripts/ab_kernels.py $W gram
  TRON_B200_DENSE_GRAM=0 timeout 900 python scripts/ab_kernels.py $W traversal
done 2>&1 | grep '^{' | tee gpurun_out/s14_ab.txt
timeout 300 python scripts/solve_wall.py P1 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8
