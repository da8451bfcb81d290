b() { timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), 'e2e', round(d['e2e']['value']), d['roundtrip_max_err'], {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
b prio
OSPH_NO_STREAM_PRIORITY=1 b noprio
b prio2
