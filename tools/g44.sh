mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -1 gpurun_out/bench2.json | cut -c1-200
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench3.json 2> gpurun_out/bench3.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench4.json 2> gpurun_out/bench4.err
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench1.json 2> gpurun_out/bench1.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
