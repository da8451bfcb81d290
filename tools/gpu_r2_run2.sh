set -x
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_pivots_sweeps.py tests/test_gpu_experiments.py -x -q -s -m gpu > gpurun_out/r2b_new.log 2>&1
tail -30 gpurun_out/r2b_new.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2b_gpu.log 2>&1
tail -15 gpurun_out/r2b_gpu.log
