"""Run the forward N times on identical input; report bitwise agreement and round-trip error per call."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1403_4661_b200 as osp
from paper_1403_4661_b200 import gridopt
L = int(sys.argv[1]); B = int(sys.argv[2]); N = int(sys.argv[3])
p = ROOT / "tests/golden/grids" / f"grid-L{L}-uniform-condmin.txt"
grid = osp.load_grid(p) if p.exists() else gridopt.optimize_order(L)
rng = np.random.default_rng(5)
flm = rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))
s = osp.inverse_sht_batch(flm, grid)
outs = []
for i in range(N):
    st = osp.TransformStats()
    f = osp.forward_sht_batch(s, grid, check=False, stats=st)
    outs.append(f.copy())
    same = "" if i == 0 else ("identical" if np.array_equal(f, outs[1 if i > 1 else 0]) else "DIFFERS max %.3e" % np.abs(f - outs[1 if i > 1 else 0]).max())
    print(f"L={L} call {i}: rt err {np.abs(f - flm).max():.3e} factor {st.extra['factor_seconds']*1e3:.1f} ms {same}", flush=True)
