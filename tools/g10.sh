mkdir -p gpurun_out
timeout 300 python tools/diag_large.py 1024 1 2>&1 | grep -v "^m=" > gpurun_out/d1.txt; cat gpurun_out/d1.txt
OSPH_FACTOR_ONE_STREAM=1 timeout 300 python tools/diag_large.py 1024 1 2>&1 | grep "call" ; 
OSPH_FACTOR_PIVOTED=1 OSPH_FACTOR_ONE_STREAM=1 timeout 300 python tools/diag_large.py 768 1 2>&1 | grep "call" ; 
OSPH_FACTOR_PIVOTED=1 timeout 300 python tools/diag_large.py 600 1 2>&1 | grep "call" ; 
timeout 900 python -m pytest tests/test_gpu_large.py -q -m gpu -s > gpurun_out/pytest_large.txt 2>&1; grep -v "^$" gpurun_out/pytest_large.txt | tail -8
