set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_pivots_sweeps.py -x -q -s -m gpu > gpurun_out/r2_piv.log 2>&1
tail -30 gpurun_out/r2_piv.log
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r2_gpu.log 2>&1
tail -15 gpurun_out/r2_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
tail -3 gpurun_out/r2_smoke.log
