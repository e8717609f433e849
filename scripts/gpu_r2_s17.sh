# full suite + the driver's default bench (P1, Gram mode) + reference arm + Q1 builder bench
set -x
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s17_bench_P1.json 2> gpurun_out/s17_bench_P1.err; tail -c 2500 gpurun_out/s17_bench_P1.json; tail -3 gpurun_out/s17_bench_P1.err
timeout 900 python bench.py --workload Q1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s17_bench_Q1.json 2> gpurun_out/s17_bench_Q1.err; tail -c 1500 gpurun_out/s17_bench_Q1.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -c 1 -o gpurun_out/P1_gram -f python scripts/profile_n1.py P1 > gpurun_out/ncu_P1_gram.log 2>&1; tail -2 gpurun_out/ncu_P1_gram.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_pass -c 1 -o gpurun_out/P1_fwd -f python scripts/profile_n1.py P1 > gpurun_out/ncu_P1_fwd.log 2>&1; tail -2 gpurun_out/ncu_P1_fwd.log
TRON_B200_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_P1.csv python bench.py --workload P1 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; ls -la gpurun_out/launches_P1.csv
