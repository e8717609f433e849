# round-2 session 3, call 2: sanitizers, parity runs (R1/P1 full, K1 eps sweep, Q1 full)
set -x
mkdir -p gpurun_out/san
timeout 300 python scripts/sanitize_cases.py > gpurun_out/san/plain.log 2>&1; tail -3 gpurun_out/san/plain.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/san/$tool.log
done
timeout 300 python scripts/parity_run.py R1 --out gpurun_out/parity_R1.json > gpurun_out/parity_R1.log 2>&1; tail -c 600 gpurun_out/parity_R1.log
timeout 600 python scripts/parity_run.py P1 --out gpurun_out/parity_P1.json > gpurun_out/parity_P1.log 2>&1; tail -c 1500 gpurun_out/parity_P1.log
timeout 900 python scripts/parity_run.py K1 --no-ref --gpu-eps 1e-3 1e-4 1e-5 1e-6 1e-8 --out gpurun_out/parity_K1_sweep.json > gpurun_out/parity_K1_sweep.log 2>&1; tail -c 2500 gpurun_out/parity_K1_sweep.log
timeout 1800 python scripts/parity_run.py Q1 --out gpurun_out/parity_Q1.json > gpurun_out/parity_Q1.log 2>&1; tail -c 2500 gpurun_out/parity_Q1.log
free -g
