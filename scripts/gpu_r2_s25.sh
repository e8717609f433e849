set -x
TRON_BENCH_WATCHDOG=100 timeout 200 python bench.py --gpus 2 --comm host --workload R1 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s25_R1_x2.json 2> gpurun_out/s25_R1_x2.err; tail -c 300 gpurun_out/s25_R1_x2.json
head -60 gpurun_out/hang_rank0.txt; head -60 gpurun_out/hang_rank1.txt
