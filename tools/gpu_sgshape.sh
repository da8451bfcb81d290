# GEMM sweep CTA tile shape (rows x maps) and stages: config 3 per variant
for v in "32x8 4" "32x8 6" "64x4 4" "64x4 6" "32x8 4" "32x8 6" "64x4 4" "64x4 6"; do set -- $v
  echo "shape=$1 stages=$2 $(OSPH_SG_SHAPE=$1 OSPH_SG_STAGES=$2 timeout 300 python bench.py --config 3 --no-cpu 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["stage_ms"]["sweep"],3), d["roundtrip_max_err"])')"; done
