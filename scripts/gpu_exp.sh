#!/bin/bash
# Kernel-time A/B of alternative library builds (build/<name>/libtron_b200.so) on workloads.
cd "$(dirname "$0")/.."
for W in ${@:-N1}; do
  echo "default $W $(timeout 600 python scripts/profile_n1.py $W 2>&1 | tail -1)"
  for V in ${VARIANTS:-exp1}; do
    echo "$V $W $(TRON_B200_LIB=$PWD/build/$V/libtron_b200.so timeout 600 python scripts/profile_n1.py $W 2>&1 | tail -1)"
  done
done
