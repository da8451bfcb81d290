"""Benchmark: fwd+inv SHT transforms/s (fp64) on the L^2-sample grid.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

Metric (BASELINE.json): forward+inverse transforms per second, whole job.  One
"transform" = one map taken through inverse_sht then forward_sht (a round
trip); a step = one inverse + one forward over a batch of B maps.  Default
workload = BASELINE configs[1]: L=256, B=64 complex fp64 maps, flm ~ complex
N(0,1) * sqrt(C_l), C_l = 1/(l(l+1)), C_0 = 1, on the reference's
condition-minimised L=256 grid.  Inputs are seeded synthetic data of that
shape/distribution (no dataset exists for this path).

Multi-GPU (N > 1, torchrun): maps are independent, so every rank runs its own
batch of B maps ("scaling": "weak"); no collective on the data path.  Timing
is CUDA events on the launching stream, max over ranks.

--impl reference times the CPU implementation of the same path: the oracle
port of the reference (oracle/, C + numpy/scipy exactly as optisph does it) on
the box's host cores, a bounded sample of maps per step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fwd+inv SHT transforms/s (fp64)"
UNIT = "transforms/s"
FP64_PEAK_TFLOPS = 37.15  # measured DMMA.8x8x4 issue rate on this pool's B200 (profiles/fp64_peak_r01.txt)

CONFIGS = {
    1: dict(L=64, B=1, spectrum="white", real=False, grid="grid-L64-uniform-condmin.txt"),
    2: dict(L=256, B=64, spectrum="cmb", real=False, grid="grid-L256-uniform-condmin.txt"),
    3: dict(L=512, B=256, spectrum="cmb", real=True, grid="grid-L512-uniform-condmin.txt"),
    4: dict(L=2048, B=1, spectrum="white", real=False, grid="grid-L2048-uniform-condmin.txt"),
    5: dict(L=4096, B=8, spectrum="cmb", real=False, grid="grid-L4096-uniform-condmin.txt"),
}


def make_coefficients(L: int, B: int, seed: int, spectrum: str, real: bool) -> np.ndarray:
    """BASELINE recipes: per map Re[L^2] then Im[L^2] ~ N(0,1), l^2+l+m order."""
    rng = np.random.default_rng(seed)
    n = L * L
    ells = np.floor(np.sqrt(np.arange(n))).astype(np.int64)
    ms = np.arange(n) - ells * ells - ells
    out = np.empty((B, n), dtype=np.complex128)
    for b in range(B):
        f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        if real:
            f[ms == 0] = f[ms == 0].real
            neg = np.nonzero(ms < 0)[0]
            pos = ells[neg] ** 2 + ells[neg] - ms[neg]
            sgn = np.where((-ms[neg]) % 2 == 1, -1.0, 1.0)
            f[neg] = sgn * np.conj(f[pos])
        if spectrum == "cmb":
            cl = np.ones(n)
            nz = ells >= 1
            cl[nz] = 1.0 / (ells[nz] * (ells[nz] + 1.0))
            f = f * np.sqrt(cl)
        out[b] = f
    return out


# ---------------------------------------------------------------------------
# algorithmic work, used for the roofline fields


def flops(L: int, B: int) -> dict:
    """Dense algorithmic fp64 flop counts per step (complex-map count)."""
    ring_fft = sum(5.0 * (2 * k + 1) * np.log2(2 * k + 1) for k in range(1, L))
    f_inv = 4.0 * B * L**3 + 1.5 * L**3 + B * ring_fft
    f_lu = sum((2.0 / 3.0) * n**3 for n in range(1, L + 1))
    f_fwd = f_lu + (8.0 / 3.0) * B * L**3 + (4.0 / 3.0) * B * L**3 + 1.5 * L**3 + B * ring_fft
    return {
        "inverse": f_inv,
        "forward": f_fwd,
        "synth": 8.0 * B * L * L * (L + 1) / 2.0,  # Legendre GEMM: 2 flops x 4B columns per (k, m, l)
        "factor_lu": sum((2.0 / 3.0) * n**3 for n in range(1, L + 1)),  # LU of every P_m
        "factor_gj": sum(2.0 * n**3 for n in range(1, L + 1)),  # executed: explicit inverse per order
        "sweep": sum(2.0 * 4 * B * ((L - m) ** 2 + m * (L - m)) for m in range(L)),
    }


# ncu DRAM traffic of the dominant kernel (one `ncu --set full` capture of the same
# workload, summarised under profiles/ by tools/ncu_summary.py), bytes per launch

NCU_PROFILES = {  # (stage, L, B) -> summary file (a multi-kernel stage sums its kernels of one call)
    ("sweep", 256, 64): "launches_r03_c2_summary.txt",
    ("factor", 256, 64): "launches_r03_c2_summary.txt",
    ("sweep", 512, 256): "launches_r03_c3_summary.txt",
    ("factor", 512, 256): "launches_r03_c3_summary.txt",
    ("factor", 2048, 1): "launches_r02_c4_summary.txt",
}


def ncu_traffic(stage: str, L: int, B: int):
    """DRAM bytes of one call's kernels of `stage`, from the committed ncu launch list summary
    (tools/launch_summary.py: lines `factor_chain_dram_bytes N` / `sweep_stage_dram_bytes N`)."""
    name = NCU_PROFILES.get((stage, L, B))
    if not name or not (ROOT / "profiles" / name).exists():
        return None, None
    key = {"factor": "factor_chain_dram_bytes", "sweep": "sweep_stage_dram_bytes"}.get(stage)
    for line in (ROOT / "profiles" / name).read_text().splitlines():
        parts = line.split()
        if len(parts) == 2 and parts[0] == key:
            return float(parts[1]), (f"profiles/{name} (dram__bytes_read.sum + dram__bytes_write.sum of the "
                                     f"{stage} stage's launches in one forward call, ncu launch list)")
    return None, None


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port of the reference)


_W = {}  # per-process worker state of the CPU arm (grid, warmed caches)


def _cpu_init(grid_path):
    """Pool initializer: load the oracle and the grid once per worker process."""
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    # a forked worker inherits BLAS pools already sized to every core: the env
    # vars come too late for them, so cap them through the libraries' own API
    # (one BLAS thread per process; 16 processes must not oversubscribe the host)
    from threadpoolctl import threadpool_limits

    _W["blas_limit"] = threadpool_limits(limits=1)
    from oracle import optisph_oracle as O

    _, _, thetas = O.load_grid_file(grid_path)
    _W["O"], _W["thetas"] = O, thetas


def _cpu_worker(args):
    L, seed, spectrum, real, grid_path, nmaps = args
    if "O" not in _W:
        _cpu_init(grid_path)
    O, thetas = _W["O"], _W["thetas"]
    flm = make_coefficients(L, nmaps, seed, spectrum, real)
    t0 = time.perf_counter()
    for b in range(nmaps):
        s = O.inverse_sht(flm[b], thetas)
        O.forward_sht(s, thetas, method="direct", check=False)  # the reference benchmark's protocol
    return nmaps, time.perf_counter() - t0


def cpu_round_trip_estimate(cfg: dict) -> tuple[float, str]:
    """Seconds per map round trip of the oracle port on one core, for L too large to time whole.

    A bounded sample, scaled up (SURVEY 8(d) "CPU baseline protocol"):
    * inverse: the reference's synthesis on 8 evenly spaced rings
      (oracle.inverse_rings, same C kernels), x L/8 -- every ring costs O(L^2);
    * forward: one order of _forward_direct (legendre_table, ring analysis,
      the gelsy solve, the k < m correction and ring update; the reference
      benchmark's method) timed at 6 orders spread over n = L - m, a cubic in
      n fitted through them and summed over all L orders.
    """
    from threadpoolctl import threadpool_limits

    from oracle import optisph_oracle as O

    O.build()
    L = cfg["L"]
    _, _, thetas = O.load_grid_file(str(ROOT / "tests" / "golden" / "grids" / cfg["grid"]))
    rng = np.random.default_rng(5)
    with threadpool_limits(limits=1):
        flm = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
        rings = [int(k) for k in np.linspace(0, L - 1, 8)]
        t0 = time.perf_counter()
        O.inverse_rings(flm, thetas, rings)
        t_inv = (time.perf_counter() - t0) * L / len(rings)
        buf = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
        roots = O.ring_roots_flat(L)
        lib = O._clib()
        ns = sorted({max(1, int(round(L * f))) for f in (1 / 32, 1 / 16, 1 / 8, 1 / 4, 1 / 2, 1.0)})
        ts = []
        for n in ns:  # one order of _forward_direct (transform.py:415-429), as the reference benchmark runs it
            m = L - n
            t0 = time.perf_counter()
            table = O.legendre_table(m, thetas, L)
            g_p = np.empty(n, dtype=np.complex128)
            g_n = np.empty(n, dtype=np.complex128)
            lib.oracle_peel_analyze(O._p(buf), O._p(roots), m, L, O._p(g_p), O._p(g_n))
            f_p, f_n = O._solve_pair(2.0 * np.pi * table[m:], g_p, g_n, m, 1.0, False)
            if m:
                cols = np.column_stack([f_p.real, f_p.imag, f_n.real, f_n.imag])
                gg = 2.0 * np.pi * (table[:m] @ cols)
                big_gp = np.ascontiguousarray(gg[:, 0] + 1j * gg[:, 1])
                big_gn = np.ascontiguousarray(gg[:, 2] + 1j * gg[:, 3])
                lib.oracle_peel_update(O._p(buf), O._p(roots), m, m, O._p(big_gp), O._p(big_gn))
            ts.append(time.perf_counter() - t0)
    coef = np.polyfit(np.array(ns, float), np.array(ts), 3)
    t_fwd = float(np.clip(np.polyval(coef, np.arange(1, L + 1, dtype=float)), 0.0, None).sum())
    how = (f"oracle port, 1 core, L={L}: inverse timed on 8 rings x L/8 ({t_inv:.2f} s/map); forward per-order "
           f"work timed at n={ns}, cubic fit summed over L orders ({t_fwd:.2f} s/map); extrapolated")
    return t_inv + t_fwd, how


class CpuPool:
    """The CPU arm's worker processes, created once (outside every timed step).

    Each worker loads the oracle, its C kernels and the grid in its initializer;
    the warm-up steps then fill the per-process caches (packed recurrence
    tables, ring roots) before any step is timed."""

    def __init__(self, cfg: dict, procs: int):
        import multiprocessing as mp

        from oracle import optisph_oracle as O

        O.build()
        self.cfg, self.procs = cfg, procs
        self.grid_path = str(ROOT / "tests" / "golden" / "grids" / cfg["grid"])
        self.pool = None
        if procs > 1:
            self.pool = mp.get_context("fork").Pool(procs, initializer=_cpu_init, initargs=(self.grid_path,))
        else:
            _cpu_init(self.grid_path)

    def run(self, maps_per_proc: int, seed: int) -> tuple[float, float]:
        """(maps, wall seconds) for procs x maps_per_proc round trips on the warm workers."""
        cfg = self.cfg
        jobs = [(cfg["L"], seed + i, cfg["spectrum"], cfg["real"], self.grid_path, maps_per_proc)
                for i in range(self.procs)]
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_worker, jobs, chunksize=1) if self.pool else [_cpu_worker(jobs[0])]
        wall = time.perf_counter() - t0
        return float(sum(r[0] for r in res)), wall

    def close(self):
        if self.pool:
            self.pool.close()
            self.pool.join()


def cpu_round_trips(cfg: dict, procs: int, maps_per_proc: int, seed: int) -> tuple[float, float]:
    """(maps, wall seconds) for procs processes x maps_per_proc round trips each (one warm-up first)."""
    pool = CpuPool(cfg, procs)
    try:
        pool.run(1, seed + 10_000)  # warm: JIT-free C kernels, but per-process tables and page faults
        return pool.run(maps_per_proc, seed)
    finally:
        pool.close()


# ---------------------------------------------------------------------------


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    maps_per_proc = 1
    times = []
    total_maps = 0.0
    pool = CpuPool(cfg, procs)  # created once, outside the timed steps; warmed by the warm-up steps
    for step in range(args.warmup + args.steps):
        maps, wall = pool.run(maps_per_proc, seed=14034661 + 100 * step)
        if step >= args.warmup:
            times.append(wall)
            total_maps += maps
    pool.close()
    value = total_maps / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(cfg, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": f"{procs} processes x {maps_per_proc} map round trip(s) per step on a pool "
                                   f"created and warmed before timing (oracle port: C kernels + "
                                   f"numpy.fft + scipy gelsy, 1 thread each)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg, args):
    return {"workload": f"L={cfg['L']}, B={cfg['B']} {'real' if cfg['real'] else 'complex'} fp64 maps, "
                        f"{'sqrt(C_l)-scaled' if cfg['spectrum'] == 'cmb' else 'unit'} complex Gaussian flm, "
                        f"inverse then forward per step",
            "L": cfg["L"], "maps_per_gpu": cfg["B"], "global_batch": cfg["B"] * args.gpus,
            "grid": cfg["grid"], "parallelism": f"maps sharded over {args.gpus} GPU(s)",
            "real_maps": "two real maps per complex transform (OSPH_REAL)" if cfg["real"] else None,
            "l2": "flushed (256 MiB write) before every timed step"}


def run_ours(args, cfg):
    import torch

    import paper_1403_4661_b200 as osp

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L, B = cfg["L"], cfg["B"]
    grid = osp.load_grid(ROOT / "tests" / "golden" / "grids" / cfg["grid"])
    flm_h = make_coefficients(L, B, 14034661 + 2 + 1000 * rank, cfg["spectrum"], cfg["real"])
    flm = torch.from_numpy(flm_h).to(dev)
    samples = torch.empty_like(flm)
    back = torch.empty_like(flm)
    plan = osp.get_plan(grid, B, local)
    stream = torch.cuda.current_stream(dev)
    plan.set_stream(osp.transform.torch_stream_handle(stream))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    real = bool(cfg["real"])
    kind = 1 | 2 | (4 if real else 0)  # OSPH_DEVICE | OSPH_ASYNC (| OSPH_REAL: two real maps per complex transform)

    def step():
        plan.inverse_raw(B, flm.data_ptr(), samples.data_ptr(), kind)
        inv_launch = plan.last_launch_count()
        plan.forward_raw(B, samples.data_ptr(), back.data_ptr(), kind, False)
        return inv_launch + plan.last_launch_count()

    # correctness guard on the measured data (not timed)
    step()
    torch.cuda.synchronize()
    err = (back - flm).abs().max().item()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stage_i = np.zeros(3)
    stage_f = np.zeros(3)
    total_ms = 0.0
    launches = 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            nl = step()
            ev1.record(stream)
            torch.cuda.synchronize()
            total_ms += ev0.elapsed_time(ev1)
            t6 = plan.last_stage_times()
            ti, tf = t6[:3], t6[3:]
            stage_i += ti
            stage_f += tf
            launches += nl
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * B * args.steps / (total_ms * 1e-3)

    # e2e: public API with pinned host buffers, H2D + D2H inside the timed region
    flm_pin = torch.from_numpy(flm_h).pin_memory()
    s_pin = torch.empty_like(flm_pin).pin_memory()
    b_pin = torch.empty_like(flm_pin).pin_memory()
    fn, sn, bn = flm_pin.numpy(), s_pin.numpy(), b_pin.numpy()
    osp.inverse_sht_batch(fn, grid, out=sn, device=local, real=real)
    osp.forward_sht_batch(sn, grid, out=bn, check=False, device=local, real=real)
    e2e_t = []
    for _ in range(max(1, min(args.steps, 5))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        osp.inverse_sht_batch(fn, grid, out=sn, device=local, real=real)
        osp.forward_sht_batch(sn, grid, out=bn, check=True, device=local, real=real)
        e2e_t.append(time.perf_counter() - t0)
    e2e_err = float(np.abs(bn - fn).max())
    if world > 1:
        t = torch.tensor([float(np.mean(e2e_t))], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_mean = float(t.item())
    else:
        e2e_mean = float(np.mean(e2e_t))
    e2e_value = world * B / e2e_mean

    if rank == 0:
        fl = flops(L, (B + 1) // 2 if real else B)  # real maps: algorithmic work of the paired transforms
        st_i = stage_i / args.steps
        st_f = stage_f / args.steps
        stages = {"pack": st_i[0], "synth": st_i[1], "ring_inverse": st_i[2],
                  "ring_forward": st_f[0], "factor": st_f[1], "sweep": st_f[2]}
        # the factor is counted as SURVEY 8(d) counts it (LU, sum 2/3 n^3), not by the
        # 3x larger work the explicit Gauss-Jordan inverse executes
        alg = {"synth": fl["synth"], "factor": fl["factor_lu"], "sweep": fl["sweep"]}

        def roof_of(stage):
            achieved = alg[stage] / stages[stage] / 1e12
            traffic, tsrc = ncu_traffic(stage, L, B)
            return {"bound": "tensor", "kernel": stage, "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                    "traffic_source": tsrc, "stage_ms": stages[stage] * 1e3,
                    "peak_source": "own fp64 DMMA microbenchmark (MEASURED_PEAKS.json has no fp64 entry)",
                    "work_count": ("SURVEY 8(d) dense count" + (": factor = sum 2/3 n^3 (LU); the kernels "
                                   "execute the explicit inverse, 3x that" if stage == "factor" else ""))}

        # The factorisation runs on side streams BESIDE the inverse and the ring DFTs of the
        # same step (it needs no data), so its stage time is wall time under sharing, not a
        # kernel-alone duration.  The headline roofline is the longest stage of the plan
        # stream's chain (pack, synth, ring DFTs, sweep -- what the step's time is made of
        # once the factors are there) when that stage has a flop count; every DMMA stage,
        # the factor included, is listed under roofline_stages.
        chain = {k: v for k, v in stages.items() if k != "factor"}
        top = max(chain, key=chain.get)
        if L > 1024:  # large single maps: the factorisation is the step (88% of it), no overlap to speak of
            top = max(stages, key=stages.get)
        roof = roof_of(top) if top in alg else None
        roof_stages = [roof_of(k) for k in ("synth", "factor", "sweep") if stages[k] > 0]
        cpu = None
        if world == 1 and not args.no_cpu and L <= 256:
            procs = 1
            maps, wall = cpu_round_trips(cfg, procs, args.cpu_maps, seed=99)
            cpu = {"value": maps / wall, "unit": UNIT, "cores": procs, "kind": "port",
                   "sample": f"{args.cpu_maps} map round trip(s), L={L}, 1 core, oracle port "
                             f"(C kernels + numpy.fft + scipy gelsy), check=False as experiments.benchmark"}
        elif world == 1 and not args.no_cpu:
            t_map, how = cpu_round_trip_estimate(cfg)
            cpu = {"value": 1.0 / t_map, "unit": UNIT, "cores": 1, "kind": "port", "sample": how}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, args),
            "stage_ms": {k: v * 1e3 for k, v in stages.items()},
            "achieved_tflops": {"inverse": fl["inverse"] / (st_i.sum()) / 1e12,
                                "forward": fl["forward"] / (st_f.sum()) / 1e12},
            "roofline": roof,
            "roofline_stages": roof_stages,
            "whole_step": {"flops": fl["inverse"] + fl["forward"],
                           "achieved_tflops": (fl["inverse"] + fl["forward"]) / (ms_per_step * 1e-3) / 1e12,
                           "frac_of_fp64_peak": (fl["inverse"] + fl["forward"]) / (ms_per_step * 1e-3) / 1e12
                                                / FP64_PEAK_TFLOPS},
            "sweep_kind": plan.last_sweep_kind(),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(2 * B * L * L * 16),
                    "d2h_bytes_per_step": int(2 * B * L * L * 16)},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "roundtrip_max_err": max(err, e2e_err),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_sharded(args, cfg, mode):
    """--shard chain|factors: the transforms split over the ranks (distributed.ShardedTransform).

    chain   one batch (configs[3]: one L=2048 map) across every rank: rings split in
            the inverse, order blocks in the forward with the spectra and coefficients
            handed down the chain (NCCL send/recv), "scaling": "strong";
    factors every rank its own B maps; the per-order factorisation split by order
            blocks and all-gathered (NCCL broadcasts) instead of repeated, "weak"."""
    import torch
    import torch.distributed as dist

    import paper_1403_4661_b200 as osp
    from paper_1403_4661_b200.distributed import ShardedTransform

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L, B = cfg["L"], cfg["B"]
    if cfg["real"]:
        raise SystemExit("--shard runs complex maps (configs 1, 2, 4, 5)")
    grid = osp.load_grid(ROOT / "tests" / "golden" / "grids" / cfg["grid"])
    seed = 14034661 + 2 + (1000 * rank if mode == "factors" else 0)
    flm_h = make_coefficients(L, B, seed, cfg["spectrum"], False)
    flm = torch.from_numpy(flm_h).to(dev)
    st = ShardedTransform(grid, B, mode)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        s = st.inverse(flm)
        return st.forward(s), st.plan.last_launch_count()

    back, _ = step()
    torch.cuda.synchronize()
    err = (back - flm).abs().max().item()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    total_ms, launches = 0.0, 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            _, nl = step()
            ev1.record(stream)
            torch.cuda.synchronize()
            total_ms += ev0.elapsed_time(ev1)
            launches += nl
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    maps_per_step = B if mode == "chain" else world * B
    value = maps_per_step * args.steps / (total_ms * 1e-3)
    # e2e: pinned host input, copied in every step; result copied out
    flm_pin = torch.from_numpy(flm_h).pin_memory()
    out_pin = torch.empty_like(flm_pin).pin_memory()
    e2e_t = []
    for _ in range(max(1, min(args.steps, 5))):
        flush.fill_(1.0)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x = flm_pin.to(dev, non_blocking=True)
        s = st.inverse(x)
        out_pin.copy_(st.forward(s, check=True))
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    e2e_err = float((out_pin - flm_pin).abs().max())
    e2e_mean = float(np.mean(e2e_t))
    if world > 1:
        t = torch.tensor([e2e_mean], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_mean = float(t.item())
    if rank == 0:
        m_lo, m_hi, k_lo, k_hi = st.ranges[0]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if mode == "chain" else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": dict(workload_config(cfg, args),
                           parallelism=(f"order blocks x {world} ranks (chain: spectra + coefficients handed "
                                        f"rank to rank, NCCL), rings split in the inverse" if mode == "chain" else
                                        f"maps per rank, factorisation split by order blocks over {world} ranks "
                                        f"and all-gathered (NCCL)"),
                           global_batch=maps_per_step),
            "shard": {"mode": mode, "rank0_orders": [m_lo, m_hi], "rank0_rings": [k_lo, k_hi]},
            "e2e": {"value": maps_per_step / e2e_mean, "unit": UNIT,
                    "h2d_bytes_per_step": int(B * L * L * 16), "d2h_bytes_per_step": int(B * L * L * 16)},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "roundtrip_max_err": max(err, e2e_err),
        }
        print(json.dumps(line), flush=True)
    st.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-maps", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--shard", default="maps", choices=["maps", "factors", "chain"],
                    help="maps: every rank its own batch (default); factors: shared factorisation; "
                         "chain: one batch across the ranks by order blocks (configs[3])")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.shard != "maps":
        run_sharded(args, cfg, args.shard)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
