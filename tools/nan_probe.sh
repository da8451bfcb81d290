timeout 60 python tools/fwd_seq.py 256 0 8 1 16 1 2>&1 | tail -6
