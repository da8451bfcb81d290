set -x
for i in 1 2; do
  OSPH_LIB=tools/libosph_ab.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2f_ab_old$i.json 2>/dev/null
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2f_ab_new$i.json 2>/dev/null
done
for f in gpurun_out/r2f_ab_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['stage_ms']['sweep'], d['stage_ms']['factor'])"; done
ncu --query-metrics --chip gb100 > gpurun_out/ncu_query.txt 2>&1 || ncu --query-metrics > gpurun_out/ncu_query.txt 2>&1
grep -i "dmma\|pipe_fp64\|fp64" gpurun_out/ncu_query.txt | head -40
