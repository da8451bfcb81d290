# diag reciprocal reorder: correctness, factor kernel launch times, benches
for L in 200 256 1024; do timeout 300 python tools/determinism.py $L 1 2 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bf_ --csv --log-file gpurun_out/bf_launch.csv python tools/fwd_once.py 256 64 2 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/bf_launch.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
for k, v in agg.items(): print(f"{k:30s} n={len(v):4d} mean={sum(v)/len(v)/1e3:8.2f} us")
PY
for c in 2 4; do timeout 300 python bench.py --config $c --no-cpu 2>&1 | tail -1 | cut -c1-160; done
