set -x
timeout 900 python -m pytest tests/test_gpu_pivots_sweeps.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2q_par.log 2>&1
tail -3 gpurun_out/r2q_par.log
for i in 1 2 3; do
  OSPH_LIB=tools/libosph_ab.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2q_old$i.json 2>/dev/null
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2q_new$i.json 2>/dev/null
done
for f in gpurun_out/r2q_*.json; do echo -n "$f "; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); s=d['stage_ms']; print(round(d['value'],1), round(s['sweep'],4), round(s['factor'],4), d['roundtrip_max_err'])"; done
