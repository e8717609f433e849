#!/bin/bash
# compute-sanitizer over every case of scripts/sanitize_cases.py, one process
# per (tool, case) so a tool limitation on one kernel cannot hide the others.
# Summary: gpurun_out/san/summary.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/san
N=$(python scripts/sanitize_cases.py --count)
: > gpurun_out/san/summary.txt
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for i in ${CASES:-$(seq 0 $((N-1)))}; do
    log=gpurun_out/san/${tool}_$i.log
    extra=""
    [ "$tool" = synccheck ] && extra="--num-cuda-barriers 4096"
    [ "$tool" = racecheck ] && extra="--num-cuda-barriers 4096 --racecheck-report all"
    timeout 900 compute-sanitizer --tool $tool $extra --print-limit 50 python scripts/sanitize_cases.py $i > $log 2>&1
    rc=$?
    name=$(grep -E "rel_f=" $log | head -1 | cut -c1-40)
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $log | tail -1)
    echo "$tool case $i [$name] rc=$rc $summ" >> gpurun_out/san/summary.txt
  done
done
cat gpurun_out/san/summary.txt
