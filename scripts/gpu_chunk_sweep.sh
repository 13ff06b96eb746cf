# bench at several chunk sizes (1M texts)
for ct in 32768 65536 131072 262144; do
  timeout 300 python bench.py --n-texts 1000000 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --chunk-tokens $ct > gpurun_out/chunk_$ct.log 2>&1
  tail -1 gpurun_out/chunk_$ct.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('chunk', $ct, 'value', round(d['value']), {k: round(v['ms_per_step'],1) for k,v in d['kernel_profile'].items()})"
done
