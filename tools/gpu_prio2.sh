b() { timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), d['roundtrip_max_err'], {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
OSPH_BF_NMIN=128 b nmin128
OSPH_BF_NMIN=64 b nmin64
OSPH_BF_NMIN=256 b nmin256
b default
