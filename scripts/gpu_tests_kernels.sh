set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python paper_2605_01060_b200/build.py -f > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -40 > gpurun_out/t_kernels.log; cat gpurun_out/t_kernels.log
