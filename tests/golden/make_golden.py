"""Generate golden fixtures by running the REFERENCE implementation (optisph).

Run in the build container, where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Outputs (committed; nothing at test time reads /root/reference):
  tests/golden/grids/grid-L{8,16,32,64,256[,512]}-uniform-condmin.txt
      produced by optisph.make_grid(..., ordering=CONDITION_MINIMIZED)
      (sampling.py:281-313, greedy optimize_order 217-278).  L=512 is copied
      from /tmp/gridgen when a previous background run of make_grid finished.
  tests/golden/grids/grid-L{16,64,256}-uniform-interleaved.txt  (sampling.py:181-208)
  tests/golden/ref_L{8,16,32,64}.npz
      thetas, flm (seeded), samples = inverse_sht(flm), fwd_direct/fwd_spectral =
      forward_sht(samples) in both methods, roundtrip error, plus legendre tables.
  tests/golden/ref_L256.npz   one map of each BASELINE input recipe at L=256 (inverse
      output + forward output) for the larger parity cases.
  tests/golden/ref_L512.npz   one real map (BASELINE configs[2] recipe) on the L=512 grid.
  tests/golden/ref_misc.npz   ring_analysis KATs, ill-conditioned order on the
      interleaved L=256 grid, legendre range cases at L=4096.
"""

import shutil
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import optisph as osp  # noqa: E402
from optisph.errors import IllConditionedSolveError  # noqa: E402

from oracle.optisph_oracle import config_coefficients  # noqa: E402

OUT = Path(__file__).resolve().parent
GRIDS = OUT / "grids"
SEED = 14034661


def grids():
    GRIDS.mkdir(exist_ok=True)
    for L in (8, 16, 32, 64, 256):
        g = osp.make_grid(L, ordering=osp.Ordering.CONDITION_MINIMIZED, cache_dir=GRIDS)
        print("condmin", L, "max kappa", max(osp.condition_number(osp.build_block(g, m)) for m in range(L)) if L <= 64 else "-")
    src512 = Path("/tmp/gridgen/grid-L512-uniform-condmin.txt")
    if src512.exists():
        shutil.copy(src512, GRIDS / src512.name)
        g = osp.load_grid(GRIDS / src512.name)
        print("condmin 512 loaded", g.band_limit)
    for L in (16, 64, 256):
        g = osp.make_grid(L)  # interleaved default
        osp.save_grid(g, GRIDS / f"grid-L{L}-uniform-interleaved.txt")


def per_L(L: int):
    grid = osp.load_grid(GRIDS / f"grid-L{L}-uniform-condmin.txt")
    rng = np.random.default_rng(SEED + L)
    flm = config_coefficients(L, rng)
    c = osp.HarmonicCoefficients(L, flm.copy())
    s = osp.inverse_sht(c, grid)
    samples = s.flatten()
    fd = osp.forward_sht(s, grid, method="direct").values
    fs = osp.forward_sht(s, grid, method="spectral").values
    # random spatial samples (Experiment 2 direction)
    rs = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
    frs = osp.forward_sht(osp.SpatialSamples.from_flat(L, rs), grid).values
    tabs = {f"table_m{m}": osp.legendre_table(m, grid.thetas, L) for m in sorted({0, 1, L // 2, L - 1})}
    np.savez_compressed(
        OUT / f"ref_L{L}.npz", thetas=grid.thetas, perm=grid.permutation, flm=flm,
        samples=samples, fwd_direct=fd, fwd_spectral=fs, rand_samples=rs,
        fwd_rand=frs, **tabs,
    )
    print(L, "E1", np.abs(fd - flm).max(), "direct-vs-spectral", np.abs(fd - fs).max())


def l256_recipes():
    grid = osp.load_grid(GRIDS / "grid-L256-uniform-condmin.txt")
    out = {}
    for name, kw in (("cmb", dict(spectrum="cmb")), ("real", dict(spectrum="cmb", real=True)),
                     ("white", dict())):
        rng = np.random.default_rng(SEED + 2)
        flm = config_coefficients(256, rng, **kw)
        s = osp.inverse_sht(osp.HarmonicCoefficients(256, flm.copy()), grid)
        f = osp.forward_sht(s, grid, method="spectral").values
        out[f"{name}_flm"] = flm
        out[f"{name}_samples"] = s.flatten()
        out[f"{name}_fwd"] = f
        print("L256", name, "E1", np.abs(f - flm).max())
    np.savez_compressed(OUT / "ref_L256.npz", thetas=grid.thetas, **out)


def misc():
    out = {}
    # ring_analysis KATs (transform.py:115-131)
    rng = np.random.default_rng(SEED)
    rings = [rng.standard_normal(2 * k + 1) + 1j * rng.standard_normal(2 * k + 1) for k in range(6)]
    ra = []
    for k, r in enumerate(rings):
        for m in range(k + 1):
            p, n = osp.ring_analysis(r, m)
            ra.append((k, m, p, n))
    out["ring_flat"] = np.concatenate(rings)
    out["ring_kat"] = np.array([(k, m, p.real, p.imag, n.real, n.imag) for k, m, p, n in ra])
    # ill-conditioned order on the (singular) interleaved L=256 grid
    g = osp.load_grid(GRIDS / "grid-L256-uniform-interleaved.txt")
    s = osp.SpatialSamples.from_flat(256, rng.standard_normal(256 * 256) + 0j)
    try:
        osp.forward_sht(s, g)
        out["illcond_order"] = np.array(-1)
    except IllConditionedSolveError as e:
        out["illcond_order"] = np.array(e.order)
        out["illcond_kappa"] = np.array(e.kappa)
        print("interleaved L256 ill-conditioned at", e.order, e.kappa)
    # legendre range (test_legendre.py:125-139 style), L=4096 near the pole
    theta = np.pi / (2 * 4096 - 1)
    for m in (0, 100, 2500, 4095):
        out[f"pole_m{m}"] = osp.legendre_table(m, [theta], 4096)[0]
    out["equator_m2000"] = osp.legendre_table(2000, [np.pi / 2], 4096)[0]
    np.savez_compressed(OUT / "ref_misc.npz", **out)


def l512_real():
    """One map of BASELINE configs[2] (real maps, sqrt(C_l)) on the reference's L=512 condmin grid."""
    grid = osp.load_grid(GRIDS / "grid-L512-uniform-condmin.txt")
    rng = np.random.default_rng(SEED + 3)
    flm = config_coefficients(512, rng, spectrum="cmb", real=True)
    s = osp.inverse_sht(osp.HarmonicCoefficients(512, flm.copy()), grid)
    f = osp.forward_sht(s, grid, method="spectral").values
    print("L512 real E1", np.abs(f - flm).max())
    np.savez_compressed(OUT / "ref_L512.npz", thetas=grid.thetas, flm=flm, samples=s.flatten(), fwd=f)


if __name__ == "__main__":
    grids()
    for L in (8, 16, 32, 64):
        per_L(L)
    l256_recipes()
    misc()
    if (GRIDS / "grid-L512-uniform-condmin.txt").exists():
        l512_real()
