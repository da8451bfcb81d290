mkdir -p gpurun_out
timeout 300 python tools/determinism.py 2048 1 3 2>&1 | tail -3
timeout 300 python tools/determinism.py 512 2 3 2>&1 | tail -3
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -1 gpurun_out/bench4.json | cut -c1-1800; tail -2 gpurun_out/bench4.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -1 gpurun_out/bench2.json | cut -c1-1500
