"""Forward transforms at (L, B) on a synthetic batch: warm-up then N timed calls (for ncu / debugging)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1403_4661_b200 as osp
L = int(sys.argv[1]); B = int(sys.argv[2]); N = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = ROOT / "tests/golden/grids" / f"grid-L{L}-uniform-condmin.txt"
grid = osp.load_grid(p) if p.exists() else osp.interleaved_grid(L)
rng = np.random.default_rng(0)
flm = rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))
s = osp.inverse_sht_batch(flm, grid)
for i in range(N):
    st = osp.TransformStats()
    f = osp.forward_sht_batch(s, grid, stats=st, check=False)
    print("fwd", i, "err %.2e" % np.abs(f - flm).max(), {k: round(v * 1e3, 3) for k, v in st.extra.items()}, flush=True)
