set -x
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2
TOOLS="memcheck" CASES="7 9 15 16" bash scripts/sanitize.sh 2>&1 | tail -4
for i in 7 9; do TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize_cases.py $i 2>&1 | grep "ERROR SUMMARY" | sed "s/^/synccheck(host) case $i: /"; done
for i in 7; do TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python scripts/sanitize_cases.py $i 2>&1 | grep "RACECHECK SUMMARY\|ERROR SUMMARY" | sed "s/^/racecheck(host) case $i: /"; done
timeout 900 python bench.py > gpurun_out/f3_P1.json 2> gpurun_out/f3_P1.err; tail -c 150 gpurun_out/f3_P1.json
timeout 1500 python bench.py --workload Q1 --steps 3 --warmup 3 > gpurun_out/f3_Q1.json 2> gpurun_out/f3_Q1.err; tail -c 150 gpurun_out/f3_Q1.json
TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1_one_solve.csv python scripts/one_solve.py P1 > /dev/null 2>&1
