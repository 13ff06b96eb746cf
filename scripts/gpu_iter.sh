# quick iteration: selected GPU tests ($1 = -k expression) + full 10M bench
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "${1:-fused}" 2>&1 | tail -30 > gpurun_out/t_iter.log; cat gpurun_out/t_iter.log
timeout 900 python bench.py --e2e-steps 1 --cpu-seconds 2 > gpurun_out/bench_iter.log 2>&1; tail -2 gpurun_out/bench_iter.log
