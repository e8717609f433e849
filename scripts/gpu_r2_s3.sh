# round-2 session 3: full GPU test suite, smoke, default bench, reference arm
set -x
nproc; free -g; lscpu | grep -E 'Model name|Socket|Core|Thread' ; nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; tail -6 gpurun_out/s3_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/s3_pytest.log 2>&1; tail -30 gpurun_out/s3_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s3_bench_P1.json 2> gpurun_out/s3_bench_P1.err
tail -c 4000 gpurun_out/s3_bench_P1.json; tail -5 gpurun_out/s3_bench_P1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s3_ref_P1.json 2>&1
tail -c 2000 gpurun_out/s3_ref_P1.json
