set -x
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6
for W in P1 Q1; do timeout 900 python scripts/ab_kernels.py $W lazy; done 2>&1 | grep '^{' | tee gpurun_out/s22_ab.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s22_bench_P1.json 2> gpurun_out/s22_bench_P1.err; tail -c 2200 gpurun_out/s22_bench_P1.json
