mkdir -p gpurun_out
for nm in 256 0; do OSPH_BF_NMIN=$nm timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('nmin=$nm', round(d['value']), round(d['roundtrip_max_err'],16), {k: round(v,3) for k,v in d['stage_ms'].items()})"; done
OSPH_BF_NMIN=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bf --csv --log-file gpurun_out/bf256_launches.csv python tools/fwd_once.py 256 64 2 > gpurun_out/ncu_bf256.log 2>&1
timeout 300 python tools/determinism.py 2048 1 2 2>&1 | tail -1
