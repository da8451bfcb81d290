"""Create, use and destroy a plan 40 times (host-buffer inverse + forward, L=256, B=32) and report
the GPU memory lost since the third iteration (0 MB expected)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1403_4661_b200 as osp  # noqa: E402
from paper_1403_4661_b200 import _lib  # noqa: E402
g = osp.load_grid(ROOT / 'tests/golden/grids/grid-L256-uniform-condmin.txt')
rng = np.random.default_rng(0)
x = rng.standard_normal((32, 256*256)) + 1j*rng.standard_normal((32, 256*256))
out = np.empty_like(x)
free0 = None
for i in range(40):
    plan = osp.transform.Plan(g.thetas, 32, 0)
    plan.inverse_raw(32, x.ctypes.data, out.ctypes.data, _lib.OSPH_HOST)
    plan.forward_raw(32, out.ctypes.data, out.ctypes.data, _lib.OSPH_HOST, True)
    plan.close()
    free, total = torch.cuda.mem_get_info()
    if i == 2: free0 = free
    if i % 10 == 9: print(i, (free0 - free) / 1e6 if free0 else 0, 'MB lost since iter 2')
print('roundtrip err', np.abs(out - x).max())
