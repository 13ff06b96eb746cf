# NEXT N1 measurements: bge-base (1M texts, 47-byte texts) and bge-large (200K texts, long texts <= 512)
timeout 900 python bench.py --encoder bgebase --n-texts 1000000 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_bgebase.log 2>&1
tail -1 gpurun_out/bench_bgebase.log | cut -c1-400
timeout 900 python bench.py --encoder bgelarge --workload long --n-texts 200000 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_bgelarge.log 2>&1
tail -1 gpurun_out/bench_bgelarge.log | cut -c1-400
