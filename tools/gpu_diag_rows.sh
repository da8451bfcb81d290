for v in 0 1; do
  if [ $v = 1 ]; then export OSPH_BF_DIAG_PATCH=1; fi
  for L in 256 512 2048; do timeout 300 python tools/determinism.py $L 2 2 2>&1 | tail -1 | sed "s/^/patch=$v /"; done
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('patch=$v cfg2', round(d['value']), d['roundtrip_max_err'], {k: round(v,3) for k,v in d['stage_ms'].items()})"
done
