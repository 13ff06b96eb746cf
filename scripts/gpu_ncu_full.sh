# ncu --set full captures of the top kernels (1M-text profile run), tags: ffn1 ffn2/ln qkv attn
set -x
mkdir -p gpurun_out
for spec in "gemm_tc_kernel<.int.256, .int.1>:ffn1:12" "gemm_tc_kernel<.int.384, .int.2>:ln:24" "gemm_tc_kernel<.int.192, .int.0>:qkv:12" "attention_window:attn:12"; do
  IFS=: read -r rx tag skip <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c 1 \
     -o gpurun_out/prof_$tag python bench.py --profile-run --n-texts 1000000 > gpurun_out/ncu_$tag.log 2>&1
  tail -n 2 gpurun_out/ncu_$tag.log
done
ls -la gpurun_out
