timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -4
timeout 60 python tools/fwd_seq.py 256 0 8 1 64 2>&1 | tail -3
timeout 60 python tools/fwd_once.py 256 64 3 2>&1 | tail -1
timeout 60 python tools/fwd_once.py 256 1 3 2>&1 | tail -1
echo fprof; OSPH_LIB=tools/libosph_fprof.so timeout 60 python tools/fwd_once.py 256 1 2 2>&1 | grep "factor_np" | sort -t= -k2 -n | tail -4
