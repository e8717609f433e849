# sanitizers on the dense cases (incremental Gram), full GPU suite, bench P1 and Q1
set -x
TOOLS="memcheck synccheck" CASES="7 9 15 16" bash scripts/sanitize.sh 2>&1 | tail -10
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s32_P1.json 2> gpurun_out/s32_P1.err; tail -c 400 gpurun_out/s32_P1.json
timeout 1200 python bench.py --workload Q1 --steps 3 --warmup 3 > gpurun_out/s32_Q1.json 2> gpurun_out/s32_Q1.err; tail -c 400 gpurun_out/s32_Q1.json; tail -n 3 gpurun_out/s32_Q1.err
