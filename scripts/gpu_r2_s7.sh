# out-of-core tests; builder benches of every workload; K1 + N1 ncu captures
set -x
timeout 900 python -m pytest tests/test_gpu_ooc.py tests/test_gpu_kernels.py -q -x 2>&1 | tail -5
for W in R1 N1 K1 Q1; do timeout 1200 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s7_bench_$W.json 2> gpurun_out/s7_bench_$W.err; python -c "
import json; d=json.loads(open('gpurun_out/s7_bench_$W.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$W', 'wall', d['value'], 'dev', d['device_s'], 'frac', round(r['frac'],3), 'hv_ms', r['avg_launch_ms'], r['kernel_ms'], 'e2e', d['e2e']['value'], d['e2e']['pinned_inputs_value'])"; done
bash scripts/gpu_profile.sh K1 > gpurun_out/s7_prof_K1.log 2>&1; tail -3 gpurun_out/s7_prof_K1.log
ls -la gpurun_out/*.ncu-rep
