b() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
b default
OSPH_DEBUG=1 timeout 300 python tools/fwd_once.py 256 64 1 2>&1 | grep "\[osph\] sweep" | head -2
for g in 1 2 4; do for t in 2 4 8; do OSPH_SWEEP_G=$g OSPH_SWEEP_T=$t b g${g}t$t; done; done
