# host-launched synccheck of the dense cases; bench P1; ncu of the delta/whole-G passes; 2-rank P1
set -x
mkdir -p gpurun_out/san_host
for i in 7 9 15 16; do
  TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 timeout 900 compute-sanitizer --tool synccheck --num-cuda-barriers 4096 --print-limit 20 python scripts/sanitize_cases.py $i > gpurun_out/san_host/synccheck_$i.log 2>&1
  echo "synccheck(host-launched) case $i: $(grep -E 'ERROR SUMMARY' gpurun_out/san_host/synccheck_$i.log | tail -1)"
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s33_P1.json 2> gpurun_out/s33_P1.err; tail -c 300 gpurun_out/s33_P1.json
TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:dense_pass_kernel --launch-count 2 -o gpurun_out/P1_fwdg_fwdd python scripts/one_solve.py P1 > gpurun_out/ncu_s33.log 2>&1; tail -2 gpurun_out/ncu_s33.log
TRON_BENCH_WATCHDOG=600 timeout 700 python bench.py --gpus 2 --comm host --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s33_P1_x2.json 2> gpurun_out/s33_P1_x2.err; tail -c 600 gpurun_out/s33_P1_x2.json; tail -n 3 gpurun_out/s33_P1_x2.err
