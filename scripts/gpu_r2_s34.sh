set -x
TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1_one_solve.csv python scripts/one_solve.py P1 > /dev/null 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s34_P1.json 2> gpurun_out/s34_P1.err; tail -c 200 gpurun_out/s34_P1.json
