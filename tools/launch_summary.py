"""Summarise an ncu launch list (CSV of gpu__time_duration.sum and DRAM bytes per launch).

Usage: python tools/launch_summary.py launches.csv "title line" > profiles/launches_rNN_summary.txt

Prints per-kernel totals and the breadth-first factor chain of the LAST
forward call (k_bf_generate .. k_bf_epilogue, plus k_kappa / k_bf_colnorm in
between) and the sweep stage after it, whose DRAM bytes bench.py reads as the
roofline traffic of those stages.  With the split factorisation the two
ranges interleave; capture launch lists with OSPH_FACTOR_SPLIT=0 so that one
chain is contiguous.
"""
import collections
import csv
import sys


def main(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, ni, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = collections.OrderedDict()
    for r in rows[1:]:
        lid = int(r[idi])
        d = launches.setdefault(lid, {"name": r[ki].split("(")[0][:44]})
        d[r[ni]] = float(r[vi].replace(",", ""))
    seq = list(launches.values())
    tot_t = sum(x.get("gpu__time_duration.sum", 0.0) for x in seq) or 1.0
    agg = collections.OrderedDict()
    for x in seq:
        a = agg.setdefault(x["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += x.get("gpu__time_duration.sum", 0.0)
        a[2] += x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)
    print(title)
    print("metrics: gpu__time_duration.sum, dram__bytes_read.sum + dram__bytes_write.sum; cold-cache, serialised launches")
    print()
    print(f"{'kernel':44s} {'n':>4s} {'total us':>10s} {'share':>7s} {'us/launch':>10s} {'DRAM MB/launch':>15s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:44s} {n:4d} {t / 1e3:10.1f} {100 * t / tot_t:6.1f}% {t / n / 1e3:10.1f} {b / n / 1e6:15.1f}")
    starts = [i for i, x in enumerate(seq) if x["name"].startswith("k_bf_generate")]
    if starts:
        i0 = starts[-1]
        i1 = i0
        while i1 < len(seq) and not seq[i1]["name"].startswith("k_bf_epilogue"):
            i1 += 1
        while i1 + 1 < len(seq) and seq[i1 + 1]["name"].startswith(("k_bf_couple", "k_kappa")):
            i1 += 1  # the coupling rows of the blocked sweep and the condition estimate close the chain
        chain = [x for x in seq[i0:i1 + 1] if x["name"].startswith(("k_bf_", "k_kappa"))]
        t = sum(x.get("gpu__time_duration.sum", 0.0) for x in chain)
        b = sum(x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0) for x in chain)
        print()
        print(f"factor chain of one forward call (k_bf_* + k_kappa, serialised): {len(chain)} launches, "
              f"{t / 1e3:.1f} us, DRAM {b / 1e6:.1f} MB")
        print(f"factor_chain_dram_bytes {int(b)}")
        # the sweep stage that follows this factor chain: every k_sb_* (blocked sweep) or
        # k_sweep* launch up to the next non-sweep kernel after the ring DFTs
        sw = [x for x in seq[i1 + 1:] if x["name"].startswith(("k_sb_", "void k_sb_", "void k_sweep", "k_fold_order0"))]
        if sw:
            t = sum(x.get("gpu__time_duration.sum", 0.0) for x in sw)
            b = sum(x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0) for x in sw)
            print(f"sweep stage of the same forward call: {len(sw)} launches, {t / 1e3:.1f} us, DRAM {b / 1e6:.1f} MB")
            print(f"sweep_stage_dram_bytes {int(b)}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
