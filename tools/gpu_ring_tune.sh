# ring DFT launch shape sweep at config 2 (RING_SMEM_KB, RING_WAVES)
b() { timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
b default
OSPH_RING_WAVES=32 b w32
OSPH_RING_WAVES=8 b w8
OSPH_RING_SMEM_KB=64 b s64
OSPH_RING_SMEM_KB=64 OSPH_RING_WAVES=32 b s64w32
