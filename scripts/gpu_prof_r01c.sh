# round-1 profile set (current) (fused QKV+attention, fused tail): full bench line, ncu launch list, --set full captures
set -x
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile-run --n-texts 1000000 > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
for spec in "mlp_tc_kernel:tail:6" "gemm_tc_kernel<.int.192, .int.4:qkvatt:6"; do
  IFS=: read -r rx tag skip <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c 1 \
     -o gpurun_out/prof_$tag python bench.py --profile-run --n-texts 1000000 > gpurun_out/ncu_$tag.log 2>&1
  tail -n 1 gpurun_out/ncu_$tag.log
done
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
