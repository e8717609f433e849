# the N > 1 bench flow on one GPU (two ranks, host data plane): P1 with parity, N1, R1
set -x
timeout 1200 python bench.py --gpus 2 --comm host --steps 3 --warmup 3 > gpurun_out/s24_P1_x2.json 2> gpurun_out/s24_P1_x2.err; tail -c 1500 gpurun_out/s24_P1_x2.json; tail -5 gpurun_out/s24_P1_x2.err
timeout 600 python bench.py --gpus 2 --comm host --workload N1 --steps 3 --warmup 3 > gpurun_out/s24_N1_x2.json 2> gpurun_out/s24_N1_x2.err; tail -c 800 gpurun_out/s24_N1_x2.json; tail -5 gpurun_out/s24_N1_x2.err
