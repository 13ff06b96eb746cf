# GPU check: parity tests, smoke, full 10M bench (scratch outputs under gpurun_out/)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/t_gpu.log; cat gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -5 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; tail -3 gpurun_out/bench_full.log
