"""Spin-weighted round trips (spin_inverse_sht + spin_forward_sht) on the GPU:
one JSON line per (L, B, spin) with device-resident throughput, end-to-end
throughput through the host-buffer API, the one-time build of the per-order
least-squares operators, stage times, kernel launches, and the oracle port's
single-core rate on a bounded sample.  Not the headline metric (BASELINE's
metric is the scalar transform); evidence for the spin row.

    python tools/bench_spin.py [--cases 64:1:2,256:64:2,512:16:1] [--steps 5] [--warmup 3]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import paper_1403_4661_b200 as osp
    from oracle import optisph_oracle as O

    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="64:1:2,256:64:2,512:16:1")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    for case in args.cases.split(","):
        L, B, s = (int(x) for x in case.split(":"))
        grid = osp.load_grid(ROOT / f"tests/golden/grids/grid-L{L}-uniform-condmin.txt")
        rng = np.random.default_rng(L + B + s)
        n = np.arange(L * L)
        ell = np.floor(np.sqrt(n)).astype(int)
        flm = rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))
        flm[:, ell < abs(s)] = 0
        plan = osp.get_plan(grid, B, 0)
        st = osp.TransformStats()
        t0 = time.perf_counter()
        samp = osp.spin_inverse_sht_batch(flm, grid, s)
        osp.spin_forward_sht_batch(samp, grid, s, stats=st)  # builds the operators
        first_wall = time.perf_counter() - t0
        build_s = st.extra["factor_seconds"]
        x = torch.from_numpy(flm).cuda()
        y = torch.empty_like(x)
        z = torch.empty_like(x)
        for _ in range(args.warmup):
            osp.spin_inverse_sht_batch(x, grid, s, out=y)
            osp.spin_forward_sht_batch(y, grid, s, out=z)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            osp.spin_inverse_sht_batch(x, grid, s, out=y)
            osp.spin_forward_sht_batch(y, grid, s, out=z, stats=st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        launches = plan.last_launch_count()
        stages = dict(zip(["pack", "synth", "ring_inverse", "ring_forward", "factor", "sweep"],
                          (float(v) * 1e3 for v in plan.last_stage_times())))
        # end to end through the host-buffer API (copies inside)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            sh = osp.spin_inverse_sht_batch(flm, grid, s)
            fh = osp.spin_forward_sht_batch(sh, grid, s)
        e2e_s = (time.perf_counter() - t0) / args.steps
        err = float(np.abs(fh - flm).max())
        line = {
            "metric": "spin fwd+inv round trips/s (fp64)", "value": B / (ms * 1e-3), "unit": "transforms/s",
            "ms_per_step": ms, "steps": args.steps, "warmup": args.warmup, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"L={L}, B={B} complex maps, spin {s}, N(0,1) flm above |s|, condmin grid",
                       "L": L, "B": B, "spin": s},
            "e2e": {"value": B / e2e_s, "unit": "transforms/s", "h2d_bytes_per_step": 2 * 16 * B * L * L,
                    "d2h_bytes_per_step": 2 * 16 * B * L * L},
            "operator_build_s": build_s, "first_call_wall_s": first_wall,
            "forward_sweep_ms": st.extra.get("sweep_seconds", 0.0) * 1e3, "gpu_launches_last_forward": launches,
            "roundtrip_max_err": err, "stages": stages,
        }
        if not args.no_cpu:
            k = 1
            t0 = time.perf_counter()
            so = O.spin_inverse_sht(flm[0], grid.thetas, s)
            O.spin_forward_sht(so, grid.thetas, s, check=False)
            cpu = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": k / cpu, "unit": "transforms/s", "cores": 1, "kind": "port",
                                    "sample": f"{k} map spin round trip, L={L}, oracle port (numpy spin tables, "
                                              "C peel kernels, scipy gelsy), 1 core"}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
