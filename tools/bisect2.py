import sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1403_4661_b200 as osp
G = ROOT / "tests/golden/grids"
def grid(L): return osp.load_grid(G / f"grid-L{L}-uniform-condmin.txt")
def check(name):
    try:
        torch.cuda.synchronize(); torch.ones(4, device="cuda").sum().item(); print("ok  ", name, flush=True)
    except Exception as e:
        print("FAIL", name, e, flush=True); sys.exit(1)
mode = sys.argv[1]
L = int(sys.argv[2])
g = grid(L)
rng = np.random.default_rng(1)
flm = rng.standard_normal((1, L * L)) + 1j * rng.standard_normal((1, L * L))
s = osp.inverse_sht_batch(flm, g); check(f"inverse {L}")
if mode == "fwd":
    osp.forward_sht_batch(s, g, check=False); check(f"forward {L}")
osp.clear_plans(); check("clear_plans")
g2 = grid(64)
osp.inverse_sht_batch(np.ones((1, 64 * 64), complex), g2); check("new plan L=64")
g3 = grid(2048)
osp.inverse_sht_batch(np.ones((1, 2048 * 2048), complex), g3); check("new plan L=2048")
