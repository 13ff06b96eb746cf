for bn in 64 128 192 256; do
  NVCC_EXTRA="-DGEMM_FORCE_BN=$bn" python paper_2605_01060_b200/build.py -f > /dev/null 2>&1
  echo "BN=$bn"; timeout 200 python scripts/gemm_bench.py 2>&1 | grep -E "qkv|ffn1_bias"
done
python paper_2605_01060_b200/build.py -f > /dev/null 2>&1
