# early-gather A/B; K1 ncu with the current kernels; gpu tests touched by the panel default change
set -x
for W in N1 K1; do
  timeout 600 python scripts/ab_kernels.py $W base
  TRON_B200_LIB=build/early/libtron_b200.so timeout 600 python scripts/ab_kernels.py $W early
done 2>&1 | grep '^{' | tee gpurun_out/s11_ab.txt
timeout 600 python -m pytest tests/test_gpu_kernels.py -q 2>&1 | tail -3
bash scripts/gpu_profile.sh K1 > gpurun_out/s11_prof_K1.log 2>&1; tail -2 gpurun_out/s11_prof_K1.log
bash scripts/gpu_profile.sh N1 > gpurun_out/s11_prof_N1.log 2>&1; tail -2 gpurun_out/s11_prof_N1.log
ls -la gpurun_out/*.ncu-rep
