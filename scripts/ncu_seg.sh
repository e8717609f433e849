#!/bin/bash
# One ncu --set full capture (with source) of the segmented transposed kernel on a workload.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
W=${1:-N1}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${2:-seg_spmv} -s ${SKIP:-3} -c 1 \
  -o gpurun_out/${W}_${2:-seg_spmv} -f python scripts/profile_n1.py $W > gpurun_out/ncu_${W}_seg.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_${W}_seg.log
