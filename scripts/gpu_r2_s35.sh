set -x
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:dense_pass_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/P1_fwdd2 python scripts/one_solve.py P1 > /dev/null 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s35_P1.json 2> gpurun_out/s35_P1.err; tail -c 200 gpurun_out/s35_P1.json
