timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for tn in 64 128 256; do echo "TN=$tn"; OSPH_SYNTH_TN=$tn timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k: round(v,4) for k,v in d['stage_ms'].items()})"; done
