#!/bin/bash
# ncu evidence for one workload: full captures of the Hv kernels + the launch list.
cd "$(dirname "$0")/.."
W=${1:-N1}
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:csr_dv -c 1 -o gpurun_out/${W}_csrdv -f python scripts/profile_n1.py $W > gpurun_out/ncu_${W}_1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:seg_spmv -s 1 -c 1 -o gpurun_out/${W}_seg -f python scripts/profile_n1.py $W > gpurun_out/ncu_${W}_2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:seg_fixup -s 1 -c 1 -o gpurun_out/${W}_fixup -f python scripts/profile_n1.py $W > gpurun_out/ncu_${W}_3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dense_accum -s 1 -c 1 -o gpurun_out/${W}_dense -f python scripts/profile_n1.py $W > gpurun_out/ncu_${W}_4.log 2>&1
TRON_B200_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${W}.csv python bench.py --workload $W --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu_${W}.log 2>&1
echo profile done
