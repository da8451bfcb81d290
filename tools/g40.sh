for r in 0 1; do OSPH_REFINE=$r timeout 300 python tools/determinism.py 2048 1 2 2>&1 | tail -1 | sed "s/^/refine=$r /"; done
OSPH_REFINE=1 timeout 300 python tools/determinism.py 1024 1 2 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_large.py -q -m gpu -s 2>&1 | grep -E "round trip|random|passed|failed"
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), {k: round(v,2) for k,v in d['stage_ms'].items()}, d['roundtrip_max_err'])"
