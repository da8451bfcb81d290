timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench.txt 2>&1; tail -1 gpurun_out/bench.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['stage_ms'])"
