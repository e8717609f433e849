# final sanitizer sweep: memcheck over every case; racecheck and synccheck host-launched on a sparse and a dense subset
set -x
TOOLS="memcheck" bash scripts/sanitize.sh 2>&1 | tail -18
for i in 0 2 3 4 7 11 15; do
  TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 python scripts/sanitize_cases.py $i > gpurun_out/san/race_host_$i.log 2>&1
  echo "racecheck(host) case $i: $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY' gpurun_out/san/race_host_$i.log | tail -1)"
  TRON_B200_DEVICE_LOOP=0 TRON_B200_NO_GRAPH=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python scripts/sanitize_cases.py $i > gpurun_out/san/sync_host_$i.log 2>&1
  echo "synccheck(host) case $i: $(grep -E 'ERROR SUMMARY' gpurun_out/san/sync_host_$i.log | tail -1)"
done
