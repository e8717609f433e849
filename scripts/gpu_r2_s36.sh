# re-run the full-size parity records with the shipped code (incremental Gram): P1, Q1, R1
set -x
timeout 1500 python scripts/parity_run.py Q1 --threads 16 --out profiles/parity_Q1.json > gpurun_out/s36_Q1.log 2>&1; tail -5 gpurun_out/s36_Q1.log
timeout 600 python scripts/parity_run.py P1 --threads 16 --out profiles/parity_P1.json > gpurun_out/s36_P1.log 2>&1; tail -5 gpurun_out/s36_P1.log
timeout 600 python scripts/parity_run.py R1 --threads 16 --out profiles/parity_R1.json > gpurun_out/s36_R1.log 2>&1; tail -3 gpurun_out/s36_R1.log
mkdir -p gpurun_out/parity && cp profiles/parity_Q1.json profiles/parity_P1.json profiles/parity_R1.json gpurun_out/parity/
