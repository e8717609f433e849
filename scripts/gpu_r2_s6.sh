# wall-time breakdown; sanitizers with/without PDL after the barrier fixes; shard test
set -x
timeout 300 python scripts/solve_wall.py R1 N1 P1 2>&1 | tail -8
timeout 600 python -m pytest tests/test_gpu_shards.py tests/test_gpu_device_loop.py tests/test_gpu_kernels.py -q -x 2>&1 | tail -4
TOOLS="synccheck racecheck" bash scripts/sanitize.sh > /dev/null 2>&1; mv gpurun_out/san/summary.txt gpurun_out/san/summary_pdl.txt; cat gpurun_out/san/summary_pdl.txt
mkdir -p gpurun_out/san_nopdl; TRON_B200_PDL=0 TOOLS="synccheck racecheck" bash scripts/sanitize.sh > /dev/null 2>&1; cp gpurun_out/san/summary.txt gpurun_out/san/summary_nopdl.txt; cat gpurun_out/san/summary_nopdl.txt
