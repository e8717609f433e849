# csr row products: NG=1 vs NG=2 groups in flight per lane (N1, K1)
set -x
for W in N1 K1; do
  python scripts/ab_kernels.py $W ng1 >> gpurun_out/s31_ab.jsonl
  TRON_B200_LIB=build/variants/libtron_ng2.so python scripts/ab_kernels.py $W ng2 >> gpurun_out/s31_ab.jsonl
done
cat gpurun_out/s31_ab.jsonl
