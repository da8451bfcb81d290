"""Per-launch list (ncu CSV of gpu__time_duration.sum + DRAM bytes) from the last k_bf_epilogue on, with per-kernel totals."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, ni, vi, idi, gi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
L = collections.OrderedDict()
for r in rows[1:]:
    d = L.setdefault(int(r[idi]), {"name": r[ki][:44], "grid": r[gi]})
    d[r[ni]] = float(r[vi].replace(",", ""))
seq = list(L.values())
pref = next((a for a in sys.argv[2:] if not a.startswith("-")), "k_bf_epilogue")
i0 = [i for i, x in enumerate(seq) if x["name"].startswith(pref)][-1]
agg = collections.OrderedDict()
for x in seq[i0:]:
    t = x.get("gpu__time_duration.sum", 0) / 1e3
    mb = (x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)) / 1e6
    if "-v" in sys.argv:
        print(f'{x["name"]:44s} {x["grid"]:>16s} {t:8.1f} us {mb:8.1f} MB')
    a = agg.setdefault(x["name"], [0, 0.0])
    a[0] += 1
    a[1] += t
for k, (n, t) in agg.items():
    print(f"{k:44s} n={n:4d} total {t:8.1f} us  avg {t / n:7.1f}")
