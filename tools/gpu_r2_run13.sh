for v in wf3 wf4; do
  OSPH_LIB=tools/libosph_$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2m_$v.json 2>/dev/null
done
OSPH_RING_WFFT=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2m_off.json 2>/dev/null
for f in gpurun_out/r2m_*.json; do echo -n "$f "; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); s=d['stage_ms']; print(round(d['value'],1), round(s['ring_inverse'],4), round(s['ring_forward'],4))"; done
