#!/bin/bash
# Full verification pass: smoke, GPU tests, bench lines for the default + dense workloads.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for W in ${@:-N1 R1 P1}; do timeout 900 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/bench_$W.log 2>&1; tail -1 gpurun_out/bench_$W.log | head -c 400; echo; done
