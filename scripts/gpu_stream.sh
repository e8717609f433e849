#!/bin/bash
# streamed segmented kernels: GPU tests, A/B vs the chunk-plan kernels, one ncu capture
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for W in N1 R1; do
  echo "$W stream  $(timeout 300 python scripts/profile_n1.py $W 2>&1 | tail -1)"
  echo "$W chunked $(TRON_B200_SEG_STREAM=0 timeout 300 python scripts/profile_n1.py $W 2>&1 | tail -1)"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:seg_stream -s 3 -c 3 -o gpurun_out/N1_stream -f python scripts/profile_n1.py N1 > gpurun_out/ncu_N1_stream.log 2>&1
echo ncu rc=$?
