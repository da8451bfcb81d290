"""One small case per code path, for compute-sanitizer (tools/sanitize.sh).

    compute-sanitizer --tool memcheck python tools/sanitize_case.py <case>

Cases: persistent (L=64, B=4: pivot discovery, breadth-first factor, persistent
sweep, Bluestein + direct rings), large (two-kernel sweep), gemm (GEMM sweep),
windowed (factor storage in windows), real (paired real maps), chain (a
multi-device plan over [0, 0]: ring-split inverse, order-block chain),
factors (multi-device batch: shared factorisation).
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1403_4661_b200 as osp  # noqa: E402
from paper_1403_4661_b200 import _lib  # noqa: E402

case = sys.argv[1]
L = int(os.environ.get("SAN_L", "64"))
grid = osp.load_grid(ROOT / "tests" / "golden" / "grids" / f"grid-L{L}-uniform-condmin.txt")
env = {"large": {"OSPH_SWEEP_LARGE": "1"}, "gemm": {"OSPH_SWEEP_GEMM": "1"},
       "windowed": {"OSPH_WINDOW_GB": "0.005"}}.get(case, {})
os.environ.update(env)
B = {"persistent": 4, "large": 2, "gemm": 16, "windowed": 2, "real": 3, "chain": 1, "factors": 4}[case]
rng = np.random.default_rng(1)
flm = rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))
devices = [0, 0] if case in ("chain", "factors") else None
plan = osp.transform.Plan(grid.thetas, B, 0, devices=devices)
kind = _lib.OSPH_HOST | (_lib.OSPH_REAL if case == "real" else 0)
if case == "real":
    from oracle import optisph_oracle as O

    flm = np.stack([O.config_coefficients(L, rng, real=True) for _ in range(B)])
s = np.empty_like(flm)
f = np.empty_like(flm)
plan.inverse_raw(B, flm.ctypes.data, s.ctypes.data, kind)
for _ in range(2):
    plan.forward_raw(B, s.ctypes.data, f.ctypes.data, kind, True)
err = np.abs(f - flm).max()
print(f"{case}: L={L} B={B} sweep={plan.last_sweep_kind() if devices is None else 'multi-device'} "
      f"round trip {err:.2e}")
plan.close()
assert err < 1e-10
