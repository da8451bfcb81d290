mkdir -p gpurun_out
timeout 300 python tools/determinism.py 2048 1 4 2>&1 | tail -4
OSPH_FACTOR_ONE_STREAM=1 timeout 300 python tools/determinism.py 2048 1 4 2>&1 | tail -4
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/determinism.py 2048 1 3 2>&1 | tail -3
timeout 300 python tools/determinism.py 1024 1 4 2>&1 | tail -4
OSPH_FACTOR_IDENTITY_PIV=1 timeout 300 python tools/determinism.py 1024 1 2 2>&1 | tail -2
OSPH_FACTOR_IDENTITY_PIV=1 timeout 300 python tools/determinism.py 512 1 2 2>&1 | tail -2
OSPH_FACTOR_IDENTITY_PIV=1 timeout 300 python tools/determinism.py 2048 1 2 2>&1 | tail -2
