# NEXT N1 measurements: bge-base (1M texts, 47-byte texts), bge-large (1M short texts; 200K long texts <= 512)
mkdir -p gpurun_out
timeout 900 python bench.py --encoder bgebase --n-texts 1000000 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_bgebase.log 2>&1
tail -1 gpurun_out/bench_bgebase.log | cut -c1-300
timeout 900 python bench.py --encoder bgelarge --n-texts 1000000 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_bgelarge_short.log 2>&1
tail -1 gpurun_out/bench_bgelarge_short.log | cut -c1-300
timeout 900 python bench.py --encoder bgelarge --workload long --n-texts 200000 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_bgelarge_long.log 2>&1
tail -1 gpurun_out/bench_bgelarge_long.log | cut -c1-300
