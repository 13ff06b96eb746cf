# bge-large long-text (C4) bench for each varlib/*.so
for so in varlib/*.so; do
  n=$(basename $so .so)
  SURGE_LIB=$so timeout 900 python bench.py --encoder bgelarge --workload long --n-texts 200000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/c4_$n.log 2>&1
  echo "$n $(tail -1 gpurun_out/c4_$n.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"]) for k,v in d["kernel_profile"].items()})')"
done
