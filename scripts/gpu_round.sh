# full GPU check: parity tests, smoke, short bench (scratch outputs under gpurun_out/)
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/t_gpu.log; cat gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -5 gpurun_out/smoke.log
timeout 600 python bench.py --n-texts 1000000 --steps 2 --warmup 1 --e2e-steps 1 --cpu-seconds 3 > gpurun_out/bench_small.log 2>&1; tail -5 gpurun_out/bench_small.log
