# fused R hand-off: determinism / round trip, GPU tests, bench configs 2-4
for L in 64 200 256 512 1024 2048; do timeout 300 python tools/determinism.py $L 1 2 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 2 3 4; do timeout 300 python bench.py --config $c 2>&1 | tail -1; done
