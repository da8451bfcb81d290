mkdir -p gpurun_out
for B in 16 64 128 256; do OSPH_DEBUG=1 timeout 300 python tools/fwd_once.py 512 $B 2 2>&1 | grep -v Warn | tail -3; done > gpurun_out/l512.txt 2>&1
cat gpurun_out/l512.txt
