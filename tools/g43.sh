timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "L512_batched or real" 2>&1 | tail -1
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['value']), {k: round(v,2) for k,v in d['stage_ms'].items()}, d['roundtrip_max_err'])"
