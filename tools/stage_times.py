"""Stage times of the device-resident inverse and forward at (L, B), every stage alone.

    OSPH_FACTOR_INLINE=1 python tools/stage_times.py L B [reps]

With OSPH_FACTOR_INLINE=1 the factorisation runs on the plan stream instead of
beside the ring DFTs, so the six stage times (CUDA events inside the library)
are those of each stage running alone; the L2 is flushed before every call."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1403_4661_b200 as osp  # noqa: E402

L, B = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
p = ROOT / "tests/golden/grids" / f"grid-L{L}-uniform-condmin.txt"
grid = osp.load_grid(p) if p.exists() else osp.interleaved_grid(L)
rng = np.random.default_rng(0)
flm = torch.from_numpy(rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))).cuda()
s = torch.empty_like(flm)
back = torch.empty_like(flm)
plan = osp.get_plan(grid, B, 0)
plan.set_stream(osp.transform.torch_stream_handle(torch.cuda.current_stream()))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
acc = np.zeros(6)
for i in range(reps + 2):
    flush.fill_(1.0)
    plan.inverse_raw(B, flm.data_ptr(), s.data_ptr(), 3)
    torch.cuda.synchronize()
    flush.fill_(1.0)
    plan.forward_raw(B, s.data_ptr(), back.data_ptr(), 3, False)
    torch.cuda.synchronize()
    if i >= 2:
        acc += plan.last_stage_times()
names = ["pack", "synth", "ring_inverse", "ring_forward", "factor", "sweep"]
print(f"L={L} B={B} err={float((back - flm).abs().max()):.2e} " +
      " ".join(f"{n}={1e3 * v / reps:.4f}ms" for n, v in zip(names, acc)))
