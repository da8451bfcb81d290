"""GPU grid optimiser vs the reference's condmin grids (L=64, 256, 512), plus eigh timing at large n."""
import sys, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1403_4661_b200 import gridopt, sampling
for L in [int(a) for a in sys.argv[1:]] or [64, 256, 512]:
    t = time.time()
    g = gridopt.optimize_order(L)
    dt = time.time() - t
    ref = sampling.load_grid(ROOT / f"tests/golden/grids/grid-L{L}-uniform-condmin.txt")
    diff = np.nonzero(g.permutation != ref.permutation)[0]
    print(f"L={L}: {dt:.1f} s, identical={diff.size == 0}, first differing ring={diff.max() if diff.size else None}", flush=True)
for n in (1024, 2048, 4096):
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    G = A.T @ A
    torch.linalg.eigh(G); torch.cuda.synchronize()
    t = time.time(); d, V = torch.linalg.eigh(G); torch.cuda.synchronize(); te = time.time() - t
    t = time.time(); torch.linalg.svd(A[:-1]); torch.cuda.synchronize(); ts = time.time() - t
    print(f"n={n}: eigh {te:.3f} s, svd {ts:.3f} s", flush=True)
