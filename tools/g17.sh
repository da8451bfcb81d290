mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "windowed" > gpurun_out/pytest_win.txt 2>&1; tail -5 gpurun_out/pytest_win.txt
timeout 1500 python tools/determinism.py 4096 1 2 > gpurun_out/det4096.txt 2>&1; tail -5 gpurun_out/det4096.txt
