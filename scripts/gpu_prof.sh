# Profile set of one round (run under gpurun on ONE GPU): the full bench line, the ncu launch list of a
# 1M-text profile run (per-launch device times; compare SHARES), and one `ncu --set full` capture of
# each hot kernel class; then scripts/ncu_summary.py writes profiles/<round>/ncu_summary.md and
# profiles/ncu_summary.json (read by bench.py for roofline.traffic).
#   bash scripts/gpu_prof.sh r02
set -x
R=${1:-r02}
mkdir -p gpurun_out profiles/$R
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 400 gpurun_out/bench_full.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile-run --n-texts 1000000 > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
for spec in "mlp_tc_kernel:tail:6" "gemm_tc_kernel<.int.192, .int.4:qkvatt:6" "embed_ln_kernel:emb:2" "meanpool_l2_kernel:pool:2" \
            "qkv_attn_tc_kernel:qkvtc:6:--att-tc 1"; do
  IFS=: read -r rx tag skip extra <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c 1 \
     -o gpurun_out/prof_$tag python bench.py --profile-run --n-texts 1000000 $extra > gpurun_out/ncu_$tag.log 2>&1
  tail -n 1 gpurun_out/ncu_$tag.log
done
python scripts/ncu_summary.py $R tail=gemm_tail qkvatt=gemm_qkv_attn emb=embed_ln pool=meanpool_l2 qkvtc=gemm_qkv_attn_tc
cp gpurun_out/launches.csv profiles/$R/launches.csv
cp gpurun_out/bench_full.json profiles/$R/bench_full.json
