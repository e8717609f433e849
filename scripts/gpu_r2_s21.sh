# Gram tiling A/B on P1 / Q1
set -x
for W in P1 Q1; do
  timeout 600 python scripts/ab_kernels.py $W base
  for v in g256 g256x2 g128x3; do TRON_B200_LIB=build/$v/libtron_b200.so timeout 600 python scripts/ab_kernels.py $W $v; done
done 2>&1 | grep '^{' | tee gpurun_out/s21_ab.txt
