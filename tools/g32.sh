timeout 300 python tools/bisect2.py inv 2048
timeout 300 python tools/bisect2.py fwd 2048
timeout 300 python tools/bisect2.py inv 4096
timeout 600 python tools/bisect2.py fwd 4096
