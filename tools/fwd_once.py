"""Inverse + forward transforms at (L, B) on a synthetic batch (for ncu captures and debugging).

    python tools/fwd_once.py L B [N]       # N forward calls after one inverse
Device-resident batches (CUDA torch tensors, one call per stage like bench.py)
unless FWD_HOST=1 (numpy: the host path copies in chunks of B/4 maps)."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1403_4661_b200 as osp  # noqa: E402

L = int(sys.argv[1])
B = int(sys.argv[2])
N = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = ROOT / "tests/golden/grids" / f"grid-L{L}-uniform-condmin.txt"
grid = osp.load_grid(p) if p.exists() else osp.interleaved_grid(L)
rng = np.random.default_rng(0)
flm = rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))
if not os.environ.get("FWD_HOST"):
    import torch

    flm = torch.from_numpy(flm).cuda()
s = osp.inverse_sht_batch(flm, grid)
for i in range(N):
    st = osp.TransformStats()
    f = osp.forward_sht_batch(s, grid, stats=st, check=False)
    err = float(abs(f - flm).max())
    print("fwd", i, "err %.2e" % err, {k: round(v * 1e3, 3) for k, v in st.extra.items()}, flush=True)
