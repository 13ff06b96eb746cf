set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -k pack -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_pack.log 2>&1; tail -1 gpurun_out/bench_pack.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["gpu_launches"], d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"],2) for k,v in d["kernel_profile"].items()})'
timeout 400 python scripts/rank_emulation.py --worlds 8 --steps 2 2>&1 | tail -1
