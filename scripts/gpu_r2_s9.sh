# LD256 default + CTA fix-ups: full suite, kernel A/B vs the previous build, bench P1/N1, synccheck without graphs
set -x
timeout 1800 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -25
for W in N1 K1; do timeout 600 python scripts/ab_kernels.py $W fixcta; done 2>&1 | grep '^{' | tee gpurun_out/s9_ab.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s9_bench_P1.json 2> gpurun_out/s9_bench_P1.err; tail -c 1500 gpurun_out/s9_bench_P1.json
timeout 600 python bench.py --workload N1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s9_bench_N1.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/s9_bench_N1.json').read().strip().splitlines()[-1]); print('N1', d['value'], d['device_s'], d['roofline']['frac'], d['clocks'])"
TRON_B200_NO_GRAPH=1 TRON_B200_DEVICE_LOOP=0 compute-sanitizer --tool synccheck python scripts/sanitize_cases.py 0 2>&1 | tail -3
TRON_B200_NO_GRAPH=1 TRON_B200_DEVICE_LOOP=0 TRON_B200_PDL=0 compute-sanitizer --tool synccheck python scripts/sanitize_cases.py 0 2>&1 | tail -3
