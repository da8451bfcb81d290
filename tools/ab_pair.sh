#!/bin/bash
# A/B: paired (rank-128) vs single (rank-64) factor steps at configs 2 and 3.
mkdir -p gpurun_out/ab
for i in 1 2 3; do
  for v in 1 0; do
    OSPH_BF_PAIR=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/ab/c2_p${v}_$i.json 2>/dev/null
    OSPH_BF_PAIR=$v timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/ab/c3_p${v}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/ab/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); s=d['stage_ms']
print('$f', round(d['value'],1), round(s['factor'],4), round(s['sweep'],4))"; done
