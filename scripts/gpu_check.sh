#!/bin/bash
# One GPU session: build check, smoke, GPU tests.  Usage: bash scripts/gpu_check.sh [pytest args]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python __graft_entry__.py 2>&1 | tail -8
timeout 1200 python -m pytest tests -q -m gpu "$@" 2>&1 | tail -60
