# the N > 1 bench flow on one GPU (two ranks over the host data plane): R1, N1, P1 (with the CPU baseline)
set -x
for W in R1 N1; do
  TRON_BENCH_WATCHDOG=240 timeout 300 python bench.py --gpus 2 --comm host --workload $W --steps 3 --warmup 3 > gpurun_out/s26_${W}_x2.json 2> gpurun_out/s26_${W}_x2.err; tail -c 600 gpurun_out/s26_${W}_x2.json; tail -3 gpurun_out/s26_${W}_x2.err
done
TRON_BENCH_WATCHDOG=600 timeout 700 python bench.py --gpus 2 --comm host --steps 3 --warmup 3 > gpurun_out/s26_P1_x2.json 2> gpurun_out/s26_P1_x2.err; tail -c 1500 gpurun_out/s26_P1_x2.json; tail -3 gpurun_out/s26_P1_x2.err
ls gpurun_out/hang_rank* 2>/dev/null && head -40 gpurun_out/hang_rank*.txt
