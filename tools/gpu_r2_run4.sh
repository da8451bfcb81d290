set -x
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -s -m gpu > gpurun_out/r2d_multi.log 2>&1
tail -30 gpurun_out/r2d_multi.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
cat gpurun_out/r2d_bench.json
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2d_bench4.json 2> gpurun_out/r2d_bench4.err
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --shard chain > gpurun_out/r2d_bench4c.json 2> gpurun_out/r2d_bench4c.err
tail -3 gpurun_out/r2d_bench4c.err
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2d_gpu.log 2>&1
tail -8 gpurun_out/r2d_gpu.log
