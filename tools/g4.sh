mkdir -p gpurun_out
OSPH_DEBUG=1 timeout 300 python tools/fwd_once.py 512 16 1 > gpurun_out/l512dbg.txt 2>&1
grep osph gpurun_out/l512dbg.txt
timeout 1200 python tools/gridopt_check.py > gpurun_out/gridopt.txt 2>&1; cat gpurun_out/gridopt.txt
