set -x
nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --workload P1 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
