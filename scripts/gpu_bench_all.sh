#!/bin/bash
# All bench lines (and the reference arm for the default workload) into gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_N1.log 2>&1
for W in ${@:-N1 R1 P1 K1 Q1}; do
  timeout 1500 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/bench_$W.log 2>&1
  echo "$W rc=$?"
done
