# memcheck over every case (Gram default, OOC, panels); final builder benches of every workload
set -x
timeout 300 python scripts/sanitize_cases.py 2>&1 | tail -16
TOOLS="memcheck" bash scripts/sanitize.sh 2>&1 | tail -16
for W in R1 N1 K1 Q1; do timeout 1500 python bench.py --workload $W --steps 5 --warmup 3 > gpurun_out/s19_bench_$W.json 2> gpurun_out/s19_bench_$W.err; tail -c 300 gpurun_out/s19_bench_$W.json; done
