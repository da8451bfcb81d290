set -x
timeout 1200 python -m pytest tests/test_gpu_variants.py -q -x -m gpu > gpurun_out/r2g_var.log 2>&1
tail -15 gpurun_out/r2g_var.log
for pr in 0 1; do
  OSPH_BF_PAIR=$pr timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2g_c2_p$pr.json 2>/dev/null
  OSPH_BF_PAIR=$pr timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2g_c4_p$pr.json 2>/dev/null
  OSPH_BF_PAIR=$pr timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2g_c3_p$pr.json 2>/dev/null
done
OSPH_LIB=tools/libosph_ab.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2g_c2_old.json 2>/dev/null
for f in gpurun_out/r2g_c*.json; do echo -n "$f "; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(round(d['value'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['roundtrip_max_err'])"; done
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2g_gpu.log 2>&1
tail -5 gpurun_out/r2g_gpu.log
