set -x
timeout 1500 python -m pytest tests/test_gpu_pivots_sweeps.py tests/test_gpu_large.py tests/test_gpu_multi.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2p_par.log 2>&1
tail -5 gpurun_out/r2p_par.log
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2p_c3.json 2>/dev/null
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2p_c4.json 2>/dev/null
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2p_c2.json 2>/dev/null
for f in gpurun_out/r2p_c*.json; do echo -n "$f "; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); s=d['stage_ms']; print(round(d['value'],3), {k: round(v,3) for k,v in s.items()}, d['roundtrip_max_err'])"; done
