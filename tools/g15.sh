mkdir -p gpurun_out
timeout 300 python tools/determinism.py 2048 1 2 2>&1 | tail -2
timeout 300 python tools/determinism.py 512 2 2 2>&1 | tail -2
timeout 300 python tools/determinism.py 1024 3 2 2>&1 | tail -2
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -1 gpurun_out/bench4.json | cut -c1-1600; tail -2 gpurun_out/bench4.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -1 gpurun_out/bench3.json | cut -c1-1600
