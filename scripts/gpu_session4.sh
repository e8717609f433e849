#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 2>&1 | tail -3
for W in N1 R1 P1; do timeout 900 python bench.py --workload $W --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_$W.log; head -c 600 gpurun_out/bench_$W.log; echo; done
bash scripts/gpu_profile.sh N1
bash scripts/gpu_profile.sh P1
