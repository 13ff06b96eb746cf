# quick GPU loop: all gpu tests + 1M-text bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/t_gpu.log; cat gpurun_out/t_gpu.log
timeout 600 python bench.py --n-texts 1000000 --steps 2 --warmup 1 --e2e-steps 1 --cpu-seconds 2 > gpurun_out/bench_small.log 2>&1; tail -1 gpurun_out/bench_small.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'e2e', d['e2e']['value']); print(d['roofline'])
[print(k, v) for k, v in d['kernel_profile'].items()]"
