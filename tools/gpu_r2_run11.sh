set -x
for kb in 48 64 96 144; do for w in 4 8 16; do
  OSPH_RING_SMEM_KB=$kb OSPH_RING_WAVES=$w timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2k_ring_${kb}_${w}.json 2>/dev/null
done; done
for f in gpurun_out/r2k_ring_*.json; do echo -n "$f "; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); s=d['stage_ms']; print(round(d['value'],1), round(s['ring_inverse'],4), round(s['ring_forward'],4))"; done
OSPH_SWEEP_NO_GEMM=1 timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2k_c3_nogemm.json 2>/dev/null
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2k_c3.json 2>/dev/null
for f in gpurun_out/r2k_c3*.json; do echo -n "$f "; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(round(d['value'],1), {k: round(v,3) for k,v in d['stage_ms'].items()})"; done
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2k_gpu.log 2>&1
tail -5 gpurun_out/r2k_gpu.log
