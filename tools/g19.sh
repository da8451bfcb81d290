mkdir -p gpurun_out
for nm in 256 128 64 0; do OSPH_BF_NMIN=$nm timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('nmin=$nm', round(d['value']), {k: round(v,3) for k,v in d['stage_ms'].items()})"; done
for nm in 256 0; do OSPH_BF_NMIN=$nm timeout 300 python tools/determinism.py 512 2 2 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "windowed" > gpurun_out/pytest_win.txt 2>&1; tail -2 gpurun_out/pytest_win.txt
