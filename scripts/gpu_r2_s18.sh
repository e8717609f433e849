# fused margin+Gram pass: tests, A/B, full suite, P1 bench
set -x
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_device_loop.py -q 2>&1 | grep -E "^E |passed|failed" | head -20
for W in P1 Q1; do
  timeout 900 python scripts/ab_kernels.py $W fused
  TRON_B200_GRAM_FUSED=0 timeout 900 python scripts/ab_kernels.py $W separate
done 2>&1 | grep '^{' | tee gpurun_out/s18_ab.txt
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s18_bench_P1.json 2> gpurun_out/s18_bench_P1.err; tail -c 600 gpurun_out/s18_bench_P1.json
