# bench each varlib/*.so twice (kernel profile), interleaved
for i in 1 2; do for so in varlib/*.so; do
  n=$(basename $so .so)
  SURGE_LIB=$so timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/vb_${n}_$i.log 2>&1
  echo "$n $i $(tail -1 gpurun_out/vb_${n}_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"]) for k,v in d["kernel_profile"].items()})')"
done; done
