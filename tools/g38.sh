for r in 0 1; do OSPH_REFINE=$r timeout 300 python tools/determinism.py 2048 1 2 2>&1 | tail -1 | sed "s/^/refine=$r /"; done
for r in 0 1; do OSPH_REFINE=$r timeout 300 python tools/determinism.py 1024 1 2 2>&1 | tail -1 | sed "s/^/refine=$r /"; done
timeout 900 python -m pytest tests/test_gpu_large.py -q -m gpu -s 2>&1 | grep -E "round trip|random|passed|failed"
