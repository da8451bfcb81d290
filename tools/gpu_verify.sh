# full GPU verification: parity tests, smoke, default bench
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', round(d['value']), 'e2e', round(d['e2e']['value']), d['roundtrip_max_err'], {k: round(v,3) for k,v in d['stage_ms'].items()})"
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['value']), d['roundtrip_max_err'], {k: round(v,2) for k,v in d['stage_ms'].items()})"
