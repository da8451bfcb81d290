set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pivots_sweeps.py -q -m gpu -x > gpurun_out/r2l_par.log 2>&1
tail -15 gpurun_out/r2l_par.log
for i in 1 2; do
  OSPH_RING_WFFT=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2l_off$i.json 2>/dev/null
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2l_on$i.json 2>/dev/null
done
for f in gpurun_out/r2l_o*.json; do echo -n "$f "; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); s=d['stage_ms']; print(round(d['value'],1), {k: round(v,4) for k,v in s.items()}, d['roundtrip_max_err'])"; done
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2l_c3.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r2l_c3.json').read().strip().splitlines()[-1]); s=d['stage_ms']; print('c3', round(d['value'],1), {k: round(v,4) for k,v in s.items()}, d['roundtrip_max_err'])"
