mkdir -p gpurun_out
timeout 1500 python tools/diag_large.py 4096 1 > gpurun_out/diag4096.txt 2>&1; cat gpurun_out/diag4096.txt
