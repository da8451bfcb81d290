mkdir -p gpurun_out
OSPH_SWEEP_LARGE=1 timeout 300 python tools/diag_large.py 256 2 > gpurun_out/diag256L.txt 2>&1; tail -4 gpurun_out/diag256L.txt
timeout 300 python tools/diag_large.py 1024 1 > gpurun_out/diag1024.txt 2>&1; cat gpurun_out/diag1024.txt
OSPH_SWEEP_LARGE=1 timeout 300 python tools/diag_large.py 1024 1 > gpurun_out/diag1024L.txt 2>&1; tail -4 gpurun_out/diag1024L.txt
timeout 600 python tools/diag_large.py 2048 1 > gpurun_out/diag2048.txt 2>&1; cat gpurun_out/diag2048.txt
OSPH_FACTOR_NO_BF=1 timeout 600 python tools/diag_large.py 512 2 > gpurun_out/diag512nobf.txt 2>&1; tail -3 gpurun_out/diag512nobf.txt
timeout 600 python tools/diag_large.py 512 2 > gpurun_out/diag512.txt 2>&1; tail -3 gpurun_out/diag512.txt
