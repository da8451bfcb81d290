mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py -q -m gpu -s > gpurun_out/pytest_large.txt 2>&1; grep -v "^$" gpurun_out/pytest_large.txt | tail -8
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -1 gpurun_out/bench3.json | cut -c1-1500; tail -2 gpurun_out/bench3.err
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -1 gpurun_out/bench4.json | cut -c1-1500; tail -2 gpurun_out/bench4.err
