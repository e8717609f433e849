#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py 2>&1 | tail -6
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -2 | tee gpurun_out/bench_n1.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:seg_spmv -s 3 -c 1 -o gpurun_out/n1_seg python scripts/profile_n1.py N1 > gpurun_out/ncu_seg.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:csr_dv -c 1 -o gpurun_out/n1_csrdv2 python scripts/profile_n1.py N1 > gpurun_out/ncu_csrdv2.log 2>&1
TRON_B200_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
echo done
