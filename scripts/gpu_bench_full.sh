# full-size bench (10M texts) + ncu launch list of a profile run (1-2 SuperBatches)
set -x
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; tail -3 gpurun_out/bench_full.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile-run --n-texts 1000000 > gpurun_out/ncu_launch.log 2>&1; tail -3 gpurun_out/ncu_launch.log
