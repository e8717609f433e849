# single-chunk segmented walk with more resident warps: A/B on N1, K1, R1
set -x
for W in N1 K1 R1; do
  timeout 600 python scripts/ab_kernels.py $W base
  TRON_B200_LIB=build/single/libtron_b200.so timeout 600 python scripts/ab_kernels.py $W single4
  TRON_B200_LIB=build/single3/libtron_b200.so timeout 600 python scripts/ab_kernels.py $W single3
done 2>&1 | grep '^{' | tee gpurun_out/s20_ab.txt
