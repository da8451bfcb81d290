"""Per-order round-trip error of the GPU spin forward against the oracle's, at a
few band limits (diagnostics for the spin sweep)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import optisph_oracle as O  # noqa: E402

import paper_1403_4661_b200 as osp  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for L in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "64,128,256").split(",")]:
    grid = osp.load_grid(ROOT / f"tests/golden/grids/grid-L{L}-uniform-condmin.txt")
    rng = np.random.default_rng(256 + s)
    n = np.arange(L * L)
    ell = np.floor(np.sqrt(n)).astype(int)
    m = n - ell * ell - ell
    flm = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
    flm[ell < abs(s)] = 0
    samp = osp.spin_inverse_sht_batch(flm[None], grid, s)[0]
    ref = O.spin_forward_sht(samp, grid.thetas, s)
    got = osp.spin_forward_sht_batch(samp[None], grid, s)[0]
    step = max(1, L // 32)
    print(f"L={L} s={s}")
    print(" ref:", " ".join("%d:%.0e" % (q, np.abs(ref - flm)[np.abs(m) == q].max()) for q in range(L - 1, -1, -step)))
    print(" gpu:", " ".join("%d:%.0e" % (q, np.abs(got - flm)[np.abs(m) == q].max()) for q in range(L - 1, -1, -step)))
    bad = [q for q in range(L - 1, -1, -1) if np.abs(got - flm)[np.abs(m) == q].max() > 1e-9]
    if bad:
        q = bad[0]
        sel = np.nonzero(np.abs(m) == q)[0]
        e = np.abs(got - flm)[sel]
        print(f" first bad order {q}: worst (l, m) = {[(int(ell[i]), int(m[i])) for i in sel[np.argsort(-e)[:6]]]}")
