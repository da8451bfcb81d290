b() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
b default
OSPH_RING_SMEM_KB=48 b smem48
OSPH_RING_SMEM_KB=160 b smem160
OSPH_RING_WAVES=8 b waves8
OSPH_RING_WAVES=16 b waves16
OSPH_RING_SMEM_KB=48 OSPH_RING_WAVES=16 b smem48w16
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -1 gpurun_out/bench5.json | cut -c1-100
