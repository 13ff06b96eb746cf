# ncu --set full of one kernel: $1 = regex, $2 = tag, $3 = launch skip
set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$1" -s ${3:-12} -c 1 \
   -o gpurun_out/prof_$2 python bench.py --profile-run --n-texts 1000000 > gpurun_out/ncu_$2.log 2>&1
tail -n 1 gpurun_out/ncu_$2.log
