"""Golden fixtures at L=4096 (BASELINE configs[4]) from the REFERENCE implementation.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_4096.py inverse   # ~15 min
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_4096.py roundtrip # after inverse
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_4096.py random
    python tests/golden/make_golden_4096.py merge

Grid: tests/golden/grids/grid-L4096-uniform-condmin.txt (this repository's GPU
greedy, gridopt.py; identical to the reference's optimize_order on every grid
the reference can produce here).  A full reference forward at L=4096 takes
hours, so the forward is the reference's own _forward_spectral loop body
(transform.py:436-467) run from m = L-1 down to M_STOP only, built from its
internals (legendre_table, _solve_pair); orders >= M_STOP depend only on orders
>= M_STOP (alias structure), so those coefficients equal the full
forward's bit for bit (verified at L=256 in the survey).

Committed slices (tests/golden/ref_L4096.npz):
  * flm = config_coefficients(4096, default_rng(SEED + 5), spectrum="cmb")
    (configs[4]: sqrt(C_l)-scaled complex Gaussian); inverse_sht(flm) on RINGS;
  * the truncated forward of those samples on orders >= M_STOP (round trip);
  * the truncated forward of complex N(0,1) samples (default_rng(SEED + 50)).
"""

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

OUT = Path(__file__).resolve().parent
L = 4096
SEED = 14034661
M_STOP = 3072
RINGS = [0, 1, 63, 64, 2047, 2048, 3000, 4095]
ORDERS = [3072, 3073, 3100, 3333, 3500, 3968, 4000, 4064, 4090, 4094, 4095]
TMP = Path("/tmp/osph_golden4096_samples.npy")


def truncated_forward(samples_flat, grid, m_stop):
    from optisph.legendre import legendre_table
    from optisph.transform import TWO_PI, SpatialSamples, _solve_pair

    s = SpatialSamples.from_flat(L, samples_flat)
    spectra = [np.fft.fft(r) for r in s.rings]
    timer = [0.0]
    out = {}
    for m in range(L - 1, m_stop - 1, -1):  # _forward_spectral body, transform.py:441-463
        table = legendre_table(m, grid.thetas, L)
        g_p = np.empty(L - m, dtype=np.complex128)
        g_n = np.empty(L - m, dtype=np.complex128)
        for k in range(m, L):
            n = 2 * k + 1
            delta = TWO_PI / n
            g_p[k - m] = delta * spectra[k][m % n]
            g_n[k - m] = delta * spectra[k][(-m) % n]
        sign = -1.0 if m % 2 else 1.0
        f_p, f_n = _solve_pair(TWO_PI * table[m:], g_p, g_n, m, sign, False, timer)
        out[m] = np.concatenate([f_p, f_n])
        if m:
            cols = np.column_stack([f_p.real, f_p.imag, f_n.real, f_n.imag])
            gg = TWO_PI * (table[:m] @ cols)
            big_gp = gg[:, 0] + 1j * gg[:, 1]
            big_gn = sign * (gg[:, 2] + 1j * gg[:, 3])
            for k in range(m):
                n = 2 * k + 1
                spectra[k][m % n] -= n * big_gp[k] / TWO_PI
                spectra[k][(-m) % n] -= n * big_gn[k] / TWO_PI
    return out


def main(part):
    from oracle.optisph_oracle import config_coefficients

    if part == "merge":
        out = {"L": L, "rings": np.array(RINGS), "orders": np.array(ORDERS), "m_stop": M_STOP}
        for p in ("inverse", "roundtrip", "random"):
            out.update(dict(np.load(OUT / f"_ref_L{L}_{p}.npz")))
        np.savez_compressed(OUT / f"ref_L{L}.npz", **out)
        print("wrote", OUT / f"ref_L{L}.npz")
        return
    import optisph as osp

    grid = osp.load_grid(OUT / "grids" / f"grid-L{L}-uniform-condmin.txt")
    t0 = time.time()
    if part == "inverse":
        flm = config_coefficients(L, np.random.default_rng(SEED + 5), spectrum="cmb")
        s = osp.inverse_sht(osp.HarmonicCoefficients(L, flm), grid)
        flat = s.flatten()
        np.save(TMP, flat)
        res = {f"inv_ring{k}": s.rings[k] for k in RINGS}
    elif part == "roundtrip":
        flat = np.load(TMP)
        f = truncated_forward(flat, grid, M_STOP)
        res = {f"rt_order{m}": f[m] for m in ORDERS}
        flm = config_coefficients(L, np.random.default_rng(SEED + 5), spectrum="cmb")
        err = 0.0
        for m, v in f.items():
            ells = np.arange(m, L)
            want = np.concatenate([flm[ells * ells + ells + m], flm[ells * ells + ells - m]])
            err = max(err, float(np.abs(v - want).max()))
        res["rt_err_top"] = np.array(err)
    elif part == "random":
        rng = np.random.default_rng(SEED + 50)
        x = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
        f = truncated_forward(x, grid, M_STOP)
        res = {f"rand_order{m}": f[m] for m in ORDERS}
    else:
        raise SystemExit(part)
    np.savez(OUT / f"_ref_L{L}_{part}.npz", **res)
    print(part, "done in %.1f s" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
