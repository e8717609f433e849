set -x
timeout 900 python -m pytest tests/test_gpu_gram.py -q -x 2>&1 | tail -2
for W in P1 Q1; do python scripts/ab_kernels.py $W ${1:-variant}; done
TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1_one_solve.csv python scripts/one_solve.py P1 > /dev/null 2>&1
