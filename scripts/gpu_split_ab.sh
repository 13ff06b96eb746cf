# tests on the in-tree library (short timeouts first: a pipeline change can hang), then an A/B of varlib/*.so
mkdir -p gpurun_out
timeout 120 python -m pytest tests -m gpu -x -q -k "mlp or tail" 2>&1 | tail -2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for so in varlib/*.so; do
  n=$(basename $so .so)
  SURGE_LIB=$so timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/vb_${n}.log 2>&1
  echo "$n $(tail -1 gpurun_out/vb_${n}.log | cut -c1-40) $(tail -1 gpurun_out/vb_${n}.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"]) for k,v in d["kernel_profile"].items()})' 2>&1 | tail -1)"
done
