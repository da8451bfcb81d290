for i in 1 2; do
  OSPH_BF_PAIR=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2o_p1_$i.json 2>/dev/null
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2o_p0_$i.json 2>/dev/null
  OSPH_SYNTH_TN=256 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2o_tn256_$i.json 2>/dev/null
done
for f in gpurun_out/r2o_*.json; do echo -n "$f "; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); s=d['stage_ms']; print(round(d['value'],1), {k: round(v,3) for k,v in s.items()})"; done
