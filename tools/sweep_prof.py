"""Run one forward transform at config 2 with the profiling build (OSPH_LIB=tools/libosph_prof.so)."""
import sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1403_4661_b200 as osp
L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
grid = osp.load_grid(ROOT / "tests/golden/grids" / f"grid-L{L}-uniform-condmin.txt") if L in (64, 256, 512) else osp.interleaved_grid(L)
rng = np.random.default_rng(0)
flm = rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))
s = osp.inverse_sht_batch(flm, grid)
st = osp.TransformStats()
f = osp.forward_sht_batch(s, grid, stats=st, check=False)
print("err", np.abs(f - flm).max(), st.extra)
for i in range(3):
    f = osp.forward_sht_batch(s, grid, stats=st, check=False)
    print("warm", i, st.extra, flush=True)
