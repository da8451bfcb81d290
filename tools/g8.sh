mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py -q -m gpu -s > gpurun_out/pytest_large.txt 2>&1; tail -15 gpurun_out/pytest_large.txt
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -1 gpurun_out/bench4.json; tail -3 gpurun_out/bench4.err
CUDA_LAUNCH_BLOCKING=1 timeout 900 python -m pytest tests -q -m gpu -x -k "real" > gpurun_out/pytest_real.txt 2>&1; tail -5 gpurun_out/pytest_real.txt
