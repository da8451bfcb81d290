"""Per-order round-trip error of the GPU forward (diagnostics for large L)."""
import sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1403_4661_b200 as osp
from paper_1403_4661_b200 import gridopt
L = int(sys.argv[1]); B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = ROOT / "tests/golden/grids" / f"grid-L{L}-uniform-condmin.txt"
grid = osp.load_grid(p) if p.exists() else gridopt.optimize_order(L)
rng = np.random.default_rng(5)
flm = rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))
s = osp.inverse_sht_batch(flm, grid)
for it in range(2):
    t = time.time()
    st = osp.TransformStats()
    f = osp.forward_sht_batch(s, grid, check=False, stats=st)
    print(f"call {it}: {time.time()-t:.2f} s", {k: round(v * 1e3, 2) for k, v in st.extra.items()},
          "max err %.3e" % np.abs(f - flm).max(), flush=True)
ells = np.floor(np.sqrt(np.arange(L * L))).astype(int)
ms = np.arange(L * L) - ells * ells - ells
err = np.abs(f - flm).max(axis=0)
for m in sorted(set([L - 1, L - 2, L - 5, L - 20, L - 100] + list(range(0, L, max(1, L // 16))))):
    if m < 0: continue
    sel = np.abs(ms) == m
    print(f"m={m:5d} max err {err[sel].max():.3e}")
print("overall", err.max())
