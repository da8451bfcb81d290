import sys, numpy as np
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import paper_1403_4661_b200 as osp
from optisph_oracle import inverse_sht
L = int(sys.argv[1]) if len(sys.argv) > 1 else 64
g = osp.load_grid(ROOT / "tests/golden/grids" / f"grid-L{L}-uniform-condmin.txt")
rng = np.random.default_rng(1)
for B in (1, 3, 20):
    flm = rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))
    s = osp.inverse_sht_batch(flm, g)
    ref = np.stack([inverse_sht(flm[b], g.thetas) for b in range(B)])
    bad = []
    for k in range(L):
        e = np.abs(s[:, k*k:(k+1)**2] - ref[:, k*k:(k+1)**2]).max()
        if e > 1e-10: bad.append((k, 2*k+1, float(e)))
    print("B", B, "bad rings", len(bad), bad[:6])
