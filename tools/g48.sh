timeout 300 python tools/determinism.py 256 3 2 2>&1 | tail -1
timeout 300 python tools/determinism.py 512 2 2 2>&1 | tail -1
timeout 300 python tools/determinism.py 1024 1 2 2>&1 | tail -1
b() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), d['roundtrip_max_err'], {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
b fused
OSPH_BF_NOFUSE=1 b nofuse
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
