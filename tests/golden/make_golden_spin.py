"""Golden fixtures of the reference's SPIN-weighted path (optisph), for the
oracle pin and the GPU parity tests of the spin transforms.

Run in the build container, where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_spin.py

Writes tests/golden/ref_spin.npz:
  seed_*         the reference's seed state _spin_seed(s, m, thetas) (mantissa,
                 offset; legendre.py:233-262) at three co-latitudes for (s, m)
                 up to band limit 4096 (exact-rational seeds)
  tab_L{L}_s{s}_m{m}   spin_table(s, m, grid.thetas, L) (legendre.py:276-306)
  L{L}_s{s}_flm / _samples / _fwd   seeded coefficients (degrees >= |s| only),
                 spin_inverse_sht of them and spin_forward_sht of those samples
                 (transform.py:474-533) on the condmin grids L = 16, 32, 64
  L16_s{s}_noise_fwd   spin_forward_sht of random (not band-limited) samples:
                 the least-squares path of the tall blocks on inconsistent data
"""

import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import optisph as osp  # noqa: E402
from optisph import legendre as leg  # noqa: E402

OUT = Path(__file__).resolve().parent
GRIDS = OUT / "grids"
SEED = 14034661


SEED_THETAS = np.array([0.3, math.pi / 2, 2.9])


def seed_rows():
    """The reference's seed state (mantissa, offset) at three co-latitudes for a
    spread of (spin, m) up to band limit 4096: pins the seed constants."""
    cases = [(s, m) for s in (-3, -2, -1, 1, 2, 3, 7) for m in range(-9, 10)]
    cases += [(s, m) for s in (1, -2, 5) for m in (100, -100, 511, -511, 1023, -1024, 2047, -3000, 4095, -4095)]
    cases += [(40, m) for m in (0, 3, -17, 39, -40, 41, 2000)]
    rows, mants, offs = [], [], []
    for s, m in cases:
        mant, off = leg._spin_seed(s, m, SEED_THETAS)
        rows.append((s, m))
        mants.append(mant)
        offs.append(off)
    return np.array(rows, dtype=np.int64), np.array(mants), np.array(offs, dtype=np.int64)


def coeffs(L, s, rng):
    n = L * L
    f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    ells = np.floor(np.sqrt(np.arange(n))).astype(np.int64)
    f[ells < abs(s)] = 0.0
    return f


def main():
    out = {}
    out["seed_rows"], out["seed_mant"], out["seed_off"] = seed_rows()
    out["seed_thetas"] = SEED_THETAS
    for L in (16, 32, 64):
        grid = osp.load_grid(GRIDS / f"grid-L{L}-uniform-condmin.txt")
        out[f"L{L}_thetas"] = grid.thetas
        for s in (1, -1, 2, 3):
            for m in (0, 1, -1, 2, -3, L // 2, -(L - 1)):
                if max(abs(m), abs(s)) < L:
                    out[f"tab_L{L}_s{s}_m{m}"] = osp.spin_table(s, m, grid.thetas, L)
            rng = np.random.default_rng(SEED + 100 * L + s)
            flm = coeffs(L, s, rng)
            c = osp.HarmonicCoefficients(L, flm.copy())
            samp = osp.spin_inverse_sht(c, grid, s)
            fwd = osp.spin_forward_sht(samp, grid, s)
            out[f"L{L}_s{s}_flm"] = flm
            out[f"L{L}_s{s}_samples"] = samp.flatten()
            out[f"L{L}_s{s}_fwd"] = fwd.values.copy()
            print(L, s, "round trip", np.abs(fwd.values - flm).max())
    grid = osp.load_grid(GRIDS / "grid-L16-uniform-condmin.txt")
    for s in (1, 2, -3):
        rng = np.random.default_rng(SEED + 7 + s)
        noise = rng.standard_normal(256) + 1j * rng.standard_normal(256)
        samp = osp.SpatialSamples.from_flat(16, noise)
        out[f"L16_s{s}_noise"] = noise
        out[f"L16_s{s}_noise_fwd"] = osp.spin_forward_sht(samp, grid, s).values.copy()
    np.savez_compressed(OUT / "ref_spin.npz", **out)
    print("wrote", OUT / "ref_spin.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
