# device-resident outer loop + host data plane shards: new tests, full suite, bench, sanitizers
set -x
timeout 600 python -m pytest tests/test_gpu_device_loop.py tests/test_gpu_shards.py -q -x 2>&1 | tail -30
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
for W in R1 N1 P1; do timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5_bench_$W.json 2> gpurun_out/s5_bench_$W.err; python -c "
import json,sys; d=json.loads(open('gpurun_out/s5_bench_$W.json').read().strip().splitlines()[-1]); print('$W', d['value'], d['device_s'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'])"; done
TOOLS="memcheck racecheck synccheck" bash scripts/sanitize.sh 2>&1 | tail -40
