# config 2 tuning knobs: breadth-first threshold and sweep ring stages
b() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
b default
OSPH_BF_NMIN=64 b nmin64
OSPH_BF_NMIN=128 b nmin128
for S in 3 5 6; do OSPH_SWEEP_S=$S b S$S; done
