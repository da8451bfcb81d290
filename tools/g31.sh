mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "not L2048_roundtrip and not gridopt" > gpurun_out/p1.txt 2>&1; echo "no-gridopt: $(tail -1 gpurun_out/p1.txt)"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/p2.txt 2>&1; echo "parity-only: $(tail -1 gpurun_out/p2.txt)"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "gridopt or large_L" > gpurun_out/p3.txt 2>&1; echo "gridopt+largeL: $(tail -1 gpurun_out/p3.txt)"
