timeout 300 python tools/determinism.py 2048 1 2 2>&1 | tail -1
timeout 300 python tools/determinism.py 512 2 2 2>&1 | tail -1
timeout 300 python tools/determinism.py 256 3 2 2>&1 | tail -1
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', round(d['value'],3), {k: round(v,2) for k,v in d['stage_ms'].items()}, d['roundtrip_max_err'])"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', round(d['value']), {k: round(v,3) for k,v in d['stage_ms'].items()})"
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['value']), {k: round(v,2) for k,v in d['stage_ms'].items()}, d['roundtrip_max_err'])"
