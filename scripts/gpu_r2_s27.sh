# incremental Gram (PM_FWDD): gram tests, P1/Q1 A/B (delta on/off), bench P1
set -x
timeout 900 python -m pytest tests/test_gpu_gram.py -x -q 2>&1 | tail -15
for W in P1 Q1; do
  for D in 1 0; do
    TRON_B200_GRAM_DELTA=$D timeout 600 python scripts/ab_kernels.py $W delta$D >> gpurun_out/s27_ab.jsonl 2> gpurun_out/s27_ab_${W}_$D.err; tail -2 gpurun_out/s27_ab_${W}_$D.err
  done
done
cat gpurun_out/s27_ab.jsonl
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s27_P1.json 2> gpurun_out/s27_P1.err; tail -c 2500 gpurun_out/s27_P1.json; tail -3 gpurun_out/s27_P1.err
