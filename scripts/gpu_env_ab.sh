# A/B of an environment switch ($1=VAR): bench with VAR=1 and VAR=0, twice, interleaved
for i in 1 2; do for v in 1 0; do
  env $1=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/envab_${v}_$i.log 2>&1
  echo "$1=$v $i $(tail -1 gpurun_out/envab_${v}_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"]) for k,v in d["kernel_profile"].items()})')"
done; done
