# A/B: fused vs separate QKV+attention on the full bench (kernel profile only)
set -x
mkdir -p gpurun_out
for f in 1 0; do
  timeout 900 python bench.py --no-e2e --no-cpu-baseline --att-fused $f > gpurun_out/bench_ab$f.log 2>&1; tail -1 gpurun_out/bench_ab$f.log | cut -c1-300
done
