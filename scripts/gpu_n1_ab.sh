# NEXT N1 encoders with the fused QKV+attention kernel on (default) and off
for f in 1 0; do
  timeout 900 python bench.py --encoder bgebase --n-texts 1000000 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --att-fused $f > gpurun_out/bench_bgebase_att$f.log 2>&1
  tail -1 gpurun_out/bench_bgebase_att$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bgebase att$f', round(d['value']), {k: round(v['ms_per_step']) for k,v in d['kernel_profile'].items()})"
done
timeout 900 python bench.py --encoder bgelarge --n-texts 300000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --att-fused 1 > gpurun_out/bench_bgelarge_short.log 2>&1
tail -1 gpurun_out/bench_bgelarge_short.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bgelarge short', round(d['value']), {k: round(v['ms_per_step']) for k,v in d['kernel_profile'].items()})"
timeout 900 python bench.py --encoder bgelarge --workload long --n-texts 200000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_bgelarge.log 2>&1
tail -1 gpurun_out/bench_bgelarge.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bgelarge long', round(d['value']), {k: round(v['ms_per_step']) for k,v in d['kernel_profile'].items()})"
