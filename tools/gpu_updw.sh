# 128-row update tiles: correctness, kernel times, benches (wide vs 64-row)
for L in 64 200 256 700 1024 2048; do timeout 300 python tools/determinism.py $L 1 2 2>&1 | tail -1; done
for rows in 128 64; do
  OSPH_BF_UPD_ROWS=$rows timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bf_update --csv --log-file gpurun_out/upd_$rows.csv python tools/fwd_once.py 1024 1 1 > /dev/null 2>&1
  python - $rows <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open(f"gpurun_out/upd_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
for k, v in agg.items(): print(sys.argv[1], f"{k:30s} n={len(v):4d} total={sum(v)/1e6:8.3f} ms")
PY
done
for c in 2 4; do for rows in 128 64; do echo rows=$rows; OSPH_BF_UPD_ROWS=$rows timeout 300 python bench.py --config $c --no-cpu 2>&1 | tail -1 | cut -c1-160; done; done
