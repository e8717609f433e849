#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/debug_dense.py 2>&1 | tee gpurun_out/debug_dense.log | tail -60
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_spmv -s 3 -c 1 -o gpurun_out/n1_merge python scripts/profile_n1.py N1 > gpurun_out/ncu_merge.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_dv -s 3 -c 1 -o gpurun_out/n1_csrdv python scripts/profile_n1.py N1 > gpurun_out/ncu_csrdv.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
tail -3 gpurun_out/ncu_merge.log
