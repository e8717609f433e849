#!/bin/bash
# A/B the dense tiled-pass configuration on P1 (tile rows x stages), then one ncu capture.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for TILE in 256 128; do for ST in 2 3 4; do
  echo "tile=$TILE stages=$ST $(TRON_B200_DENSE_TILE=$TILE TRON_B200_DENSE_STAGES=$ST timeout 300 python scripts/profile_n1.py P1 2>&1 | tail -1)"
done; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dense_pass -s 2 -c 2 -o gpurun_out/P1_dense_pass -f python scripts/profile_n1.py P1 > gpurun_out/ncu_P1_dense.log 2>&1
echo ncu rc=$?
