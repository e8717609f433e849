# validation after the one-launch Gram CG, pinned spare, sampler handshake
set -x
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TOOLS="memcheck" CASES="7 9 10 15 16" bash scripts/sanitize.sh 2>&1 | tail -5
for i in 7 15; do TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize_cases.py $i 2>&1 | grep "ERROR SUMMARY" | sed "s/^/synccheck(host) case $i: /"; done
timeout 900 python bench.py > gpurun_out/f2_P1.json 2> gpurun_out/f2_P1.err; tail -c 200 gpurun_out/f2_P1.json
timeout 900 python bench.py --impl reference > gpurun_out/f2_ref.json 2> gpurun_out/f2_ref.err; tail -c 200 gpurun_out/f2_ref.json
for W in R1 N1; do timeout 600 python bench.py --workload $W > gpurun_out/f2_$W.json 2> gpurun_out/f2_$W.err; done
timeout 1500 python bench.py --workload Q1 --steps 3 --warmup 3 > gpurun_out/f2_Q1.json 2> gpurun_out/f2_Q1.err
TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1_one_solve.csv python scripts/one_solve.py P1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f2_launches_P1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/f2_* gpurun_out/p1_one_solve.csv | wc -l
