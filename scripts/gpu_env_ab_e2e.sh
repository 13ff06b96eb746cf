# A/B of an environment switch ($1=VAR) on the e2e (streaming ABI, no per-kernel events) number
for i in 1 2; do for v in 1 0; do
  env $1=$v timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/envab_${v}_$i.log 2>&1
  echo "$1=$v $i $(tail -1 gpurun_out/envab_${v}_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), d["clocks"]["sm_mhz"])')"
done; done
