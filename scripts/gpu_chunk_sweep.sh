# chunk size sweep on the full 10M bench (kernel-profiled device path + e2e)
for c in 131072 262144 524288 1048576; do
  timeout 900 python bench.py --chunk-tokens $c --steps 2 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/chunk_$c.log 2>&1
  echo "chunk $c $(tail -1 gpurun_out/chunk_$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"]) for k,v in d["kernel_profile"].items()})')"
done
