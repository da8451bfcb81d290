# GEMM sweep cp.async stage count: config 3 bench per variant, then the GPU suite on the default
for ns in 4 3 2 4; do echo "stages=$ns $(OSPH_SG_STAGES=$ns timeout 300 python bench.py --config 3 --no-cpu 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["stage_ms"]["sweep"],3), d["roundtrip_max_err"])')"; done
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
