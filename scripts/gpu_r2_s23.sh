set -x
for W in P1 Q1; do
  timeout 600 python scripts/ab_kernels.py $W base
  TRON_B200_LIB=build/gpf/libtron_b200.so timeout 600 python scripts/ab_kernels.py $W prefetch
done 2>&1 | grep '^{' | tee gpurun_out/s23_ab.txt
