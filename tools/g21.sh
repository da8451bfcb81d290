mkdir -p gpurun_out
for nm in 256 128 0; do OSPH_BF_NMIN=$nm timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('nmin=$nm', round(d['value']), round(d['roundtrip_max_err'],16), {k: round(v,3) for k,v in d['stage_ms'].items()})"; done
timeout 300 python tools/determinism.py 2048 1 2 2>&1 | tail -1
OSPH_BF_NMIN=0 timeout 300 python tools/determinism.py 512 2 2 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
