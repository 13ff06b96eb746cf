# attention heads-per-CTA sweep (rebuilds kernels.cu with -DATT_HEADS_PER_CTA)
for hg in 1 2 4; do
  NVCC_EXTRA="-DATT_HEADS_PER_CTA=$hg" python paper_2605_01060_b200/build.py -f > /dev/null 2>&1
  timeout 300 python bench.py --n-texts 1000000 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/att_$hg.log 2>&1
  tail -1 gpurun_out/att_$hg.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('hg', $hg, 'value', round(d['value']), 'attn', round(d['kernel_profile']['attention']['ms_per_step'],1))"
done
timeout 120 python -m pytest tests/test_gpu_kernels.py -q -k attention 2>&1 | tail -1
