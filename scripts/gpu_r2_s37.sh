# transposed product: L2 priority hints (u evict_last; bases and out evict_first) A/B on K1, N1, R1
set -x
for W in K1 N1 R1; do
  python scripts/ab_kernels.py $W base >> gpurun_out/s37_ab.jsonl
  TRON_B200_LIB=build/variants/libtron_l2hint.so python scripts/ab_kernels.py $W l2hint >> gpurun_out/s37_ab.jsonl
done
cat gpurun_out/s37_ab.jsonl
