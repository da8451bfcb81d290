timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -4
timeout 60 python tools/fwd_seq.py 256 0 8 1 64 2>&1 | tail -3
OSPH_DEBUG=1 timeout 60 python tools/fwd_once.py 256 64 3 2>&1 | tail -2
OSPH_DEBUG=1 timeout 60 python tools/fwd_once.py 256 1 3 2>&1 | tail -2
timeout 120 python tools/fwd_once.py 512 8 2 2>&1 | tail -1
echo prof; OSPH_LIB=tools/libosph_prof.so timeout 60 python tools/sweep_prof.py 256 64 2>&1 | grep -i "prof" | tail -2
