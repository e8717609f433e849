#!/bin/bash
cd "$(dirname "$0")/.."
for D in 0 2; do for W in ${@:-N1 R1}; do echo "dbg=$D $W $(TRON_B200_STREAM_DEBUG=$D timeout 600 python scripts/profile_n1.py $W 2>&1 | tail -1)"; done; done
for W in ${@:-N1 R1}; do echo "chunked $W $(TRON_B200_SEG_STREAM=0 timeout 600 python scripts/profile_n1.py $W 2>&1 | tail -1)"; done
