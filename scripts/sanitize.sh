# SURVEY.md §5 auxiliaries on the GPU box:
#  (1) compute-sanitizer memcheck / racecheck / synccheck over the C1 toy path (__graft_entry__.smoke:
#      the streaming ABI, all kernels of the toy config);
#  (2) a ThreadSanitizer build of the host runtime (libsurge with -fsanitize=thread) driven by
#      scripts/tsan_driver.cpp: one submitting thread, one polling/releasing thread.
# Logs go to gpurun_out/sanitize_*.log.
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|smoke ok' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
# the round-2 kernels (tcgen05 QKV + attention, cluster-pair LN GEMMs, long-text tcgen05 attention)
for tool in memcheck synccheck; do
  for tc in 1 0; do
    SURGE_ATT_LONG_TC=$tc timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all \
      python scripts/sanitize_new_kernels.py > gpurun_out/sanitize_new_${tool}_tc$tc.log 2>&1
    echo "new kernels $tool long_tc=$tc rc=$? $(grep -E 'ERROR SUMMARY|new kernels ok' gpurun_out/sanitize_new_${tool}_tc$tc.log | tr '\n' ' ')"
  done
done
TSAN=$(gcc -print-file-name=libtsan.so)
SURGE_BUILD_OUT=varlib/tsan.so SURGE_BUILD_DIR=varlib/_b_tsan NVCC_EXTRA="-Xcompiler -fsanitize=thread,-g" \
  NVCC_LINK_EXTRA="-Xcompiler -fsanitize=thread" python paper_2605_01060_b200/build.py -f > /dev/null
g++ -O1 -g -fsanitize=thread -o varlib/tsan_driver scripts/tsan_driver.cpp varlib/tsan.so -Wl,-rpath,$PWD/varlib -lpthread
TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1" timeout 900 ./varlib/tsan_driver > gpurun_out/sanitize_tsan.log 2>&1
echo "tsan rc=$? races=$(grep -c 'WARNING: ThreadSanitizer' gpurun_out/sanitize_tsan.log) $(grep 'tsan driver' gpurun_out/sanitize_tsan.log | tr '\n' ' ')"
