# round-2 session 2: tests after the engine retirement, the new bench (P1 default)
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_P1.json 2> gpurun_out/r2_bench_P1.err
tail -c 3000 gpurun_out/r2_bench_P1.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_ref_P1.json 2>&1
cat gpurun_out/r2_ref_P1.json
