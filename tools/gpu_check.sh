set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
OSPH_DEBUG=1 timeout 120 python tools/fwd_once.py 256 64 3 2>&1 | tail -5
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.txt 2>&1; tail -2 gpurun_out/bench.txt
