# ncu --set full capture of one kernel (regex $1, output tag $2) in a profile run of the 1M-text workload
set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$1" -s ${3:-12} -c 1 \
   -o gpurun_out/prof_$2 python bench.py --profile-run --n-texts 1000000 > gpurun_out/ncu_$2.log 2>&1
tail -n 3 gpurun_out/ncu_$2.log
