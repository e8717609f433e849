#!/bin/bash
# Round-1 profile artifacts: launch lists (ncu, CG loop host-driven so kernels are visible) and
# full captures of the Hv kernels for N1 (sparse) and P1 (dense).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for W in N1 R1 P1; do
  TRON_B200_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${W}.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench_under_ncu_${W}.log 2>&1
  echo "$W launches rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"csr_dv|seg_spmv|seg_fixup" -s 3 -c 3 \
  -o gpurun_out/N1_hv -f python scripts/profile_n1.py N1 > gpurun_out/ncu_N1_hv.log 2>&1; echo "N1 full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_pass -s 2 -c 2 \
  -o gpurun_out/P1_hv -f python scripts/profile_n1.py P1 > gpurun_out/ncu_P1_hv.log 2>&1; echo "P1 full rc=$?"
