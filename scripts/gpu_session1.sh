#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/gpu_check.sh --timeout 300 2>&1 | tee gpurun_out/check.log | tail -80
timeout 600 python bench.py --steps 3 --warmup 3 2>&1 | tail -5 | tee gpurun_out/bench1.log
