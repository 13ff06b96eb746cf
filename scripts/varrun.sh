# A/B timing on one GPU: each argument is  <lib>[:<bench args>]  (lib = varlib/<lib>.so, or "head" for the
# in-tree build); prints texts/s and per-kernel-class ms per step at 2M texts.
mkdir -p gpurun_out
for spec in "$@"; do
  v=${spec%%:*}; extra=""; [[ "$spec" == *:* ]] && extra=${spec#*:}
  lib=varlib/$v.so; [ "$v" = head ] && lib=paper_2605_01060_b200/libsurge.so
  tag=$(echo "$spec" | tr ' :=' '___')
  SURGE_LIB=$lib timeout 300 python bench.py --n-texts 2000000 --no-e2e --no-cpu-baseline --steps 3 --warmup 3 $extra > gpurun_out/var_$tag.json 2> gpurun_out/var_$tag.err
  python - "$tag" <<'PY'
import json,sys
v=sys.argv[1]
try:
  d=json.loads(open(f"gpurun_out/var_{v}.json").read().strip().splitlines()[-1])
  kp=d["kernel_profile"]
  print(v, "texts/s %.0f"%d["value"], " ".join(f"{k}={kp[k]['ms_per_step']:.1f}" for k in kp), "clk", d.get("clocks",{}).get("sm_mhz"))
except Exception as e: print(v, "ERR", e, open(f"gpurun_out/var_{v}.err").read()[-800:])
PY
done
