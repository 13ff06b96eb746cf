# one GPU call: build check, parity tests, smoke, full bench, ncu launch list, ncu --set full of the top kernels
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/t_gpu.log; cat gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log | cut -c1-600
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile-run --n-texts 1000000 > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
for spec in "gemm_tc_kernel<256, 1>:ffn1:20" "attention_window:attn:8" "gemm_tc_kernel<384, 2>:ln:20" "gemm_tc_kernel<192, 0>:qkv:10"; do
  IFS=: read -r rx tag skip <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c 1 \
     -o gpurun_out/prof_$tag python bench.py --profile-run --n-texts 1000000 > gpurun_out/ncu_$tag.log 2>&1
  tail -n 2 gpurun_out/ncu_$tag.log
done
ls -la gpurun_out
