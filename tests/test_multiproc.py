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


# ---------------------------------------------------------------------------
# ShardedTransform's exchange logic (chain and factors) over gloo, with a
# host-memory plan standing in for each rank's GPU (tests/_fake_shard_plan.py)

_FAKE_L, _FAKE_B = 12, 3


class _FakeGrid:
    band_limit = _FAKE_L
    thetas = np.linspace(0.1, 3.0, _FAKE_L)


def _fake_inputs():
    rng = np.random.default_rng(11)
    n = _FAKE_L * _FAKE_L
    return [rng.standard_normal((_FAKE_B, n)) + 1j * rng.standard_normal((_FAKE_B, n)) for _ in range(2)]


def _fake_run(mode):
    import torch

    from _fake_shard_plan import FakeShardPlan
    from paper_1403_4661_b200.distributed import ShardedTransform

    flm, samples = (torch.from_numpy(a) for a in _fake_inputs())
    plan = FakeShardPlan(_FAKE_L, _FAKE_B)
    st = ShardedTransform(_FakeGrid(), _FAKE_B, mode, device="cpu", plan=plan)
    inv = st.inverse(flm).numpy()
    fwd = st.forward(samples).numpy()
    return inv, fwd, plan.stages


def _fake_worker(rank, world, port, mode, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank,) + _fake_run(mode))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,world", [("chain", 2), ("chain", 3), ("factors", 2), ("factors", 3)])
def test_sharded_transform_exchange_gloo(mode, world):
    import multiprocessing as mp

    from paper_1403_4661_b200 import _lib

    sys.path.insert(0, str(ROOT / "tests"))
    inv1, fwd1, stages1 = _fake_run(mode)  # one rank: no exchange
    assert np.isfinite(inv1).all()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fake_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=240) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, inv, fwd, stages in res:
        if mode == "chain":
            assert np.array_equal(inv, inv1)  # every rank holds every ring
            # rank 0 alone transforms the rings; every rank factors its own block
            want = _lib.STAGE_RINGS | _lib.STAGE_FACTOR if rank == 0 else _lib.STAGE_FACTOR
            assert stages == [want, _lib.STAGE_SWEEP]
        else:
            assert np.array_equal(inv, inv1)  # own maps, no exchange
            assert stages == [_lib.STAGE_FACTOR, _lib.STAGE_RINGS | _lib.STAGE_SWEEP]
        assert np.array_equal(fwd, fwd1)  # identical to the unsharded run, bit for bit
