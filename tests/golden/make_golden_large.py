"""Golden fixtures at L=2048 (BASELINE configs[3]) from the REFERENCE implementation.

Run in the build container (needs /root/reference), one part per process so
they run side by side:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_large.py inverse
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_large.py roundtrip
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_large.py random
    python tests/golden/make_golden_large.py merge

The grid is tests/golden/grids/grid-L2048-uniform-condmin.txt, produced by this
repository's GPU greedy (gridopt.py; the same greedy as optimize_order,
sampling.py:217-278, checked identical to the reference's own grids for
L <= 512) and loaded here by the reference's load_grid (crc32 verified).

Inputs are regenerated from seeds at test time, so only small slices are
committed (tests/golden/ref_L2048.npz):
  * flm = config_coefficients(2048, default_rng(SEED + 4)) (configs[3]: white
    complex N(0,1)); inverse_sht(flm) (transform.py:347-357) on the rings RINGS;
  * forward_sht(inverse_sht(flm), method="spectral") (transform.py:436-467),
    its max round-trip error over all L^2 coefficients, and its coefficients of
    the orders ORDERS;
  * samples = complex N(0,1) from default_rng(SEED + 40) (not band-limited):
    forward_sht(samples, method="spectral") on the orders ORDERS.
"""

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

OUT = Path(__file__).resolve().parent
L = 2048
SEED = 14034661
RINGS = [0, 1, 2, 3, 10, 63, 64, 255, 256, 1000, 1023, 1024, 1500, 2000, 2046, 2047]
ORDERS = [0, 1, 2, 3, 17, 100, 511, 1000, 1024, 1500, 2000, 2040, 2046, 2047]


def order_values(flm: np.ndarray, m: int) -> np.ndarray:
    ells = np.arange(abs(m), L)
    return np.concatenate([flm[ells * ells + ells + m], flm[ells * ells + ells - m]])


def main(part: str):
    from oracle.optisph_oracle import config_coefficients

    if part == "merge":
        parts = {p: dict(np.load(OUT / f"_ref_L{L}_{p}.npz")) for p in ("inverse", "roundtrip", "random")}
        out = {"L": L, "rings": np.array(RINGS), "orders": np.array(ORDERS)}
        for d in parts.values():
            out.update(d)
        np.savez_compressed(OUT / f"ref_L{L}.npz", **out)
        print("wrote", OUT / f"ref_L{L}.npz")
        return
    import optisph as osp

    grid = osp.load_grid(OUT / "grids" / f"grid-L{L}-uniform-condmin.txt")
    flm = config_coefficients(L, np.random.default_rng(SEED + 4))
    t0 = time.time()
    if part == "inverse":
        s = osp.inverse_sht(osp.HarmonicCoefficients(L, flm), grid)
        res = {f"inv_ring{k}": s.rings[k] for k in RINGS}
    elif part == "roundtrip":
        s = osp.inverse_sht(osp.HarmonicCoefficients(L, flm), grid)
        f = osp.forward_sht(s, grid, method="spectral", check=False).values
        res = {"rt_err": np.array(np.abs(f - flm).max())}
        res.update({f"rt_order{m}": order_values(f, m) for m in ORDERS})
    elif part == "random":
        rng = np.random.default_rng(SEED + 40)
        x = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
        f = osp.forward_sht(osp.SpatialSamples.from_flat(L, x), grid, method="spectral", check=False).values
        res = {f"rand_order{m}": order_values(f, m) for m in ORDERS}
        res["rand_max"] = np.array(np.abs(f).max())
    else:
        raise SystemExit(f"unknown part {part}")
    np.savez(OUT / f"_ref_L{L}_{part}.npz", **res)
    print(part, "done in %.1f s" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
