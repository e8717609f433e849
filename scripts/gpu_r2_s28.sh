# 8-warp dense pass (inline producer) + incremental Gram: dense tests, A/B vs the producer-warp build
set -x
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_kernels.py -q -k "gram or dense or svm or Dense" 2>&1 | tail -15
for W in P1 Q1; do
  timeout 600 python scripts/ab_kernels.py $W inline >> gpurun_out/s28_ab.jsonl 2> gpurun_out/s28_e1.err
  TRON_B200_LIB=build/variants/libtron_prodwarp.so timeout 600 python scripts/ab_kernels.py $W prodwarp >> gpurun_out/s28_ab.jsonl 2> gpurun_out/s28_e2.err
  TRON_B200_GRAM_DELTA=0 timeout 600 python scripts/ab_kernels.py $W inline_nodelta >> gpurun_out/s28_ab.jsonl 2> gpurun_out/s28_e3.err
done
cat gpurun_out/s28_ab.jsonl; tail -3 gpurun_out/s28_e*.err
