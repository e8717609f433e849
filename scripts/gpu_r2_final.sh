# round-end validation: GPU suite, smoke, default bench (P1), the reference arm, R1/N1/K1/Q1 lines
set -x
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/final_P1.json 2> gpurun_out/final_P1.err; tail -c 300 gpurun_out/final_P1.json
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -c 400 gpurun_out/final_ref.json
for W in R1 N1; do timeout 600 python bench.py --workload $W > gpurun_out/final_$W.json 2> gpurun_out/final_$W.err; tail -c 200 gpurun_out/final_$W.json; done
timeout 1500 python bench.py --workload K1 --steps 3 --warmup 3 > gpurun_out/final_K1.json 2> gpurun_out/final_K1.err; tail -c 200 gpurun_out/final_K1.json
timeout 1500 python bench.py --workload Q1 --steps 3 --warmup 3 > gpurun_out/final_Q1.json 2> gpurun_out/final_Q1.err; tail -c 200 gpurun_out/final_Q1.json
