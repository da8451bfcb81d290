"""Summarise an ncu --set full report (key metrics + top stall reasons + top source lines) as text."""
import collections
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    # fp64 tensor-core (DMMA) pipe: capture with
    #   --metrics sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,
    #             sm__inst_executed_pipe_tensor_subpipe_dmma.sum
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    return {k: (x, u) for k, u, x in zip(h, units, v)}


def source(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, agg, text = None, collections.Counter(), {}
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        try:
            ln = int(r[0])
            v = float(r[4])
        except (ValueError, IndexError):
            continue
        if cur and cur.endswith((".cu", ".cuh")) and not cur.startswith(("sm_", "cooperative", "helpers")):
            agg[(cur, ln)] += v
            if r[1].strip():
                text[(cur, ln)] = r[1].strip()[:90]
    return agg, text


def main(rep, title):
    d = raw(rep)
    print(title)
    print("report:", rep.split("/")[-1])
    for k in KEYS:
        if k in d:
            print(f"  {k:62s} {d[k][0]:>16s} {d[k][1]}")
    stalls = {k: float(v[0]) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v[0]}
    tot = sum(stalls.values()) or 1.0
    print("  warp-state samples (share):")
    for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:10]:
        print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:5.1f}%")
    agg, text = source(rep)
    tot = sum(agg.values()) or 1.0
    print("  top source lines (share of samples):")
    for (f, l), v in agg.most_common(15):
        print(f"    {100 * v / tot:5.1f}%  {f}:{l}  {text.get((f, l), '')}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
