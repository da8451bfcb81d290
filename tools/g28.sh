mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "legendre or gridopt" > gpurun_out/san1.txt 2>&1; grep -E "Invalid|ERROR SUMMARY|passed|failed|at 0x|by thread" gpurun_out/san1.txt | head -20
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "real" > gpurun_out/san2.txt 2>&1; grep -E "Invalid|ERROR SUMMARY|passed|failed|at 0x|by thread" gpurun_out/san2.txt | head -20
