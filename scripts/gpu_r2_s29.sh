# full GPU suite + default bench after the incremental Gram and the 8-warp dense pass
set -x
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s29_P1.json 2> gpurun_out/s29_P1.err; tail -c 3000 gpurun_out/s29_P1.json; tail -n 3 gpurun_out/s29_P1.err
