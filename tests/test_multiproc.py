"""CPU, world_size 2 over gloo: the multi-GPU host logic (map sharding, gather,
max-over-ranks timing) with the oracle standing in for each rank's GPU."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1403_4661_b200.distributed import shard_bounds

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("total,world", [(64, 2), (7, 2), (5, 8), (256, 8), (1, 2)])
def test_shard_bounds_partition(total, world):
    seen = []
    for r in range(world):
        lo, hi = shard_bounds(total, r, world)
        assert 0 <= lo <= hi <= total
        seen.extend(range(lo, hi))
    assert seen == list(range(total))
    sizes = [shard_bounds(total, r, world)[1] - shard_bounds(total, r, world)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from oracle import optisph_oracle as O
    from paper_1403_4661_b200 import load_grid
    from paper_1403_4661_b200.distributed import max_over_ranks, sharded_apply

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid = load_grid(ROOT / "tests/golden/grids/grid-L16-uniform-condmin.txt")
        rng = np.random.default_rng(5)
        B = 5
        flm = rng.standard_normal((B, 256)) + 1j * rng.standard_normal((B, 256))
        calls = []

        def compute(x):
            calls.append(x.shape[0])
            return np.stack([O.inverse_sht(v, grid.thetas) for v in x])

        out = sharded_apply(flm, compute)
        t = max_over_ranks(float(rank + 1))
        q.put((rank, out, calls, t))
    finally:
        dist.destroy_process_group()


def test_sharded_apply_two_ranks_gloo():
    import multiprocessing as mp

    from oracle import optisph_oracle as O
    from paper_1403_4661_b200 import load_grid

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    grid = load_grid(ROOT / "tests/golden/grids/grid-L16-uniform-condmin.txt")
    rng = np.random.default_rng(5)
    flm = rng.standard_normal((5, 256)) + 1j * rng.standard_normal((5, 256))
    ref = np.stack([O.inverse_sht(v, grid.thetas) for v in flm])
    res.sort(key=lambda r: r[0])
    assert res[0][2] == [3] and res[1][2] == [2]  # shard sizes 3 + 2
    for rank, out, _, t in res:
        assert np.array_equal(out, ref)  # gathered batch identical on every rank
        assert t == 2.0  # max over ranks
