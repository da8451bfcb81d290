set -x
for i in 1 2; do
  OSPH_LIB=tools/libosph_ab.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2h_old$i.json 2>/dev/null
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2h_new$i.json 2>/dev/null
done
for f in gpurun_out/r2h_*.json; do echo -n "$f "; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(round(d['value'],1), {k: round(v,4) for k,v in d['stage_ms'].items()}, d['roundtrip_max_err'])"; done
timeout 1500 python -m pytest tests/test_gpu_pivots_sweeps.py tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_variants.py -q -m gpu > gpurun_out/r2h_gpu.log 2>&1
tail -5 gpurun_out/r2h_gpu.log
