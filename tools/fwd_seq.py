"""Forward transforms at L for a sequence of batch sizes (debugging): python tools/fwd_seq.py L check B1 B2 ..."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1403_4661_b200 as osp
L = int(sys.argv[1]); check = sys.argv[2] == "1"; Bs = [int(x) for x in sys.argv[3:]]
p = ROOT / "tests/golden/grids" / f"grid-L{L}-uniform-condmin.txt"
grid = osp.load_grid(p) if p.exists() else osp.interleaved_grid(L)
rng = np.random.default_rng(0)
flm = rng.standard_normal((max(Bs), L * L)) + 1j * rng.standard_normal((max(Bs), L * L))
s = osp.inverse_sht_batch(flm, grid)
for B in Bs:
    f = osp.forward_sht_batch(s[:B], grid, check=check)
    e = np.abs(f - flm[:B])
    bad = np.argwhere(~np.isfinite(e))
    print("B", B, "check", check, "err %.2e" % np.nanmax(e), "nonfinite", len(bad), bad[:4].tolist(), flush=True)
    if len(bad):
        idx = bad[:, 1]
        ell = np.floor(np.sqrt(idx)).astype(int)
        m = idx - ell * ell - ell
        for mm in sorted(set(np.abs(m).tolist()))[::16] + [int(np.abs(m).max())]:
            sel = np.abs(m) == mm
            print("  |m|=%d: %d bad, ell in [%d, %d]" % (mm, sel.sum(), ell[sel].min(), ell[sel].max()))
        big = np.argwhere(np.isfinite(e) & (e > 1e-9))
        print("  finite but wrong:", len(big))
