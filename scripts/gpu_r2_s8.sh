# A/B of the sparse stream loads (256-bit evict_first) and L2 persistence; shard test detail; synccheck probe
set -x
for W in N1 K1; do
  timeout 600 python scripts/ab_kernels.py $W base
  TRON_B200_LIB=build/ld256/libtron_b200.so timeout 600 python scripts/ab_kernels.py $W ld256
  TRON_B200_L2_PERSIST=1 timeout 600 python scripts/ab_kernels.py $W persist
  TRON_B200_L2_PERSIST=1 TRON_B200_LIB=build/ld256/libtron_b200.so timeout 600 python scripts/ab_kernels.py $W ld256+persist
done 2>&1 | grep -E '^\{|Error|error' | tee gpurun_out/s8_ab.txt
timeout 600 python -m pytest "tests/test_gpu_shards.py::test_two_shards_compose[dense-svm]" -q -x 2>&1 | grep -E "^E |assert|passed|failed" | head -20
compute-sanitizer --tool synccheck scripts/synccheck_probe_bin 2>&1 | tail -8
