set -x
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2j_c2.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r2j_c2.json').read().strip().splitlines()[-1]); print(round(d['value'],1), {k: round(v,4) for k,v in d['stage_ms'].items()}, d['roundtrip_max_err'])"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_pivots_sweeps.py -q -m gpu -x > gpurun_out/r2j_gpu.log 2>&1
tail -3 gpurun_out/r2j_gpu.log
bash tools/profile_r02.sh > gpurun_out/r2j_prof.log 2>&1
ls gpurun_out/*.ncu-rep
bash tools/fp64_peak_clocks.sh
