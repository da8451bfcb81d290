set -x
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -s -m gpu > gpurun_out/r2c_multi.log 2>&1
tail -30 gpurun_out/r2c_multi.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
tail -2 gpurun_out/r2c_bench.err; cat gpurun_out/r2c_bench.json
timeout 900 python -m pytest tests/test_gpu_pivots_sweeps.py tests/test_gpu_parity.py -q -m gpu > gpurun_out/r2c_par.log 2>&1
tail -5 gpurun_out/r2c_par.log
