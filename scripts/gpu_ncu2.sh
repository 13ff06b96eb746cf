# ncu --set full of the FFN1 (weight-stationary BN=192) and QKV kernels after the epilogue rewrite
set -x
mkdir -p gpurun_out
python paper_2605_01060_b200/build.py > /dev/null
for spec in "gemm_tc_kernel<.int.192, .int.1, .bool.1>:ffn1ws:12" "gemm_tc_kernel<.int.192, .int.0, .bool.1>:qkvws:12" "attention_tile:attn2:12"; do
  IFS=: read -r rx tag skip <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c 1 \
     -o gpurun_out/prof_$tag python bench.py --profile-run --n-texts 1000000 > gpurun_out/ncu_$tag.log 2>&1
  tail -n 2 gpurun_out/ncu_$tag.log
done
