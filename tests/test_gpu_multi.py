"""GPU: the multi-GPU partitions against the single-GPU transforms.

The box has one B200, so the partitions are exercised with every shard on
device 0 -- which checks the partitioning and the hand-offs, not speed:

* a multi-device plan over devices [0, 0] (one process, peer copies between
  the sub-plans): a single map runs as the order-block chain (ring-split
  inverse), a batch splits its maps with the factorisation split by order
  blocks and the factors copied to every sub-plan;
* two processes (torch.distributed, gloo data plane through host memory, so
  no kernel of one rank waits on the other) running ShardedTransform in
  chain and factors mode.

The chain does, per order, exactly the kernels of the single-GPU windowed
forward (factor storage in windows of orders, window.cu), so its coefficients
must equal that forward's bit for bit; against the default single-GPU path
(the persistent sweep) they agree to rounding.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1403_4661_b200 as osp
from paper_1403_4661_b200 import _lib

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def same(a, b):
    """Bitwise equality, with the size of the difference in the failure message."""
    assert a.shape == b.shape
    assert np.array_equal(a, b), f"max |diff| {np.abs(a - b).max():.3e} (scale {np.abs(b).max():.3e})"


def _single(grid, samples, env=None, monkeypatch=None):
    if env:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
    plan = osp.transform.Plan(grid.thetas, samples.shape[0], 0)
    out = np.empty_like(samples)
    plan.forward_raw(samples.shape[0], samples.ctypes.data, out.ctypes.data, _lib.OSPH_HOST, True)
    plan.close()
    if env:
        for k in env:
            monkeypatch.delenv(k)
    return out


@pytest.mark.parametrize("L,ndev", [(64, 2), (256, 3), (1024, 2)])
def test_group_plan_chain_single_map(L, ndev, grid_of, monkeypatch):
    g = grid_of(L)  # L = 1024: the GPU greedy's grid (refinement on for L > 512)
    rng = np.random.default_rng(L + ndev)
    flm = rng.standard_normal((1, L * L)) + 1j * rng.standard_normal((1, L * L))
    ref_s = osp.inverse_sht_batch(flm, g)
    plan = osp.transform.Plan(g.thetas, 1, devices=[0] * ndev)
    s = np.empty_like(flm)
    plan.inverse_raw(1, flm.ctypes.data, s.ctypes.data, _lib.OSPH_HOST)  # ring-split inverse
    same(s, ref_s)
    f = np.empty_like(flm)
    plan.forward_raw(1, s.ctypes.data, f.ctypes.data, _lib.OSPH_HOST, True)
    plan.close()
    windowed = _single(g, s, {"OSPH_WINDOW_GB": "0.02" if L < 1024 else "1"}, monkeypatch)
    same(f, windowed)  # same per-order kernels, blocks instead of windows
    default = _single(g, s)
    assert np.abs(f - default).max() <= 1e-12 * max(1.0, np.abs(default).max())
    assert np.abs(f - flm).max() <= (1e-10 if L <= 256 else 1e-8)


@pytest.mark.parametrize("L,B,ndev", [(64, 4, 2), (256, 6, 3), (512, 4, 2)])
def test_group_plan_batch_shared_factors(L, B, ndev, grid_of):
    g = grid_of(L)
    rng = np.random.default_rng(7 * L + B)
    flm = rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))
    plan = osp.transform.Plan(g.thetas, B, devices=[0] * ndev)
    s = np.empty_like(flm)
    plan.inverse_raw(B, flm.ctypes.data, s.ctypes.data, _lib.OSPH_HOST)  # maps split
    shards = [osp.distributed.shard_bounds(B, i, ndev) for i in range(ndev)]
    # (per shard: the synthesis kernel and its tiles depend on the batch size)
    same(s, np.concatenate([osp.inverse_sht_batch(flm[b0:b1], g) for b0, b1 in shards]))
    f = np.empty_like(flm)
    for _ in range(2):  # the second call reuses the plans (pivots known, factors re-gathered)
        plan.forward_raw(B, s.ctypes.data, f.ctypes.data, _lib.OSPH_HOST, True)
    plan.close()
    # factors computed by their owners and copied: the same bits as one device factoring every order
    ref = np.concatenate([osp.forward_sht_batch(s[b0:b1], g) for b0, b1 in shards])
    same(f, ref)
    assert np.abs(f - flm).max() <= 1e-10


def test_group_plan_check_reports_failing_order(golden, grid_of):
    d = golden("ref_misc.npz")
    g = grid_of(256, "interleaved")
    s = np.random.default_rng(1).standard_normal((1, 256 * 256)) + 0j
    plan = osp.transform.Plan(g.thetas, 1, devices=[0, 0])
    out = np.empty_like(s)
    with pytest.raises(osp.IllConditionedSolveError) as err:
        plan.forward_raw(1, s.ctypes.data, out.ctypes.data, _lib.OSPH_HOST, True)
    plan.close()
    assert err.value.order == int(d["illcond_order"])


# ---------------------------------------------------------------------------
# one process per rank (torch.distributed), both ranks on GPU 0 with gloo

WORKER = r"""
import os, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import torch, torch.distributed as dist
import paper_1403_4661_b200 as osp
from paper_1403_4661_b200.distributed import ShardedTransform
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
L, mode, out = int(sys.argv[2]), sys.argv[3], sys.argv[4]
grid = osp.load_grid(sys.argv[1] + f"/tests/golden/grids/grid-L{L}-uniform-condmin.txt")
rng = np.random.default_rng(L)
if mode == "chain":
    flm = rng.standard_normal((1, L * L)) + 1j * rng.standard_normal((1, L * L))
else:  # every rank its own maps
    allm = rng.standard_normal((2 * world, L * L)) + 1j * rng.standard_normal((2 * world, L * L))
    flm = allm[2 * rank:2 * rank + 2]
st = ShardedTransform(grid, flm.shape[0], mode)
x = torch.from_numpy(flm).cuda()
s = st.inverse(x)
f = st.forward(s, check=True)
f2 = st.forward(s)  # plans reused
torch.cuda.synchronize()
np.savez(out + f".{rank}.npz", s=s.cpu().numpy(), f=f.cpu().numpy(), f2=f2.cpu().numpy(), flm=flm)
st.close()
dist.destroy_process_group()
"""


def _run_ranks(tmp_path, L, mode, world=2):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29500 + (os.getpid() % 2000)),
               WORLD_SIZE=str(world))
    procs = []
    for r in range(world):
        e = dict(env, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER, str(ROOT), str(L), mode,
                                       str(tmp_path / mode)], env=e))
    for p in procs:
        assert p.wait(timeout=900) == 0
    return [np.load(tmp_path / f"{mode}.{r}.npz") for r in range(world)]


@pytest.mark.parametrize("L", [64, 512])
def test_processes_chain(tmp_path, L, grid_of, monkeypatch):
    res = _run_ranks(tmp_path, L, "chain")
    g = grid_of(L)
    flm = res[0]["flm"]
    s_ref = osp.inverse_sht_batch(flm, g)
    windowed = _single(g, s_ref, {"OSPH_WINDOW_GB": "0.02" if L < 512 else "0.2"}, monkeypatch)
    for r in res:  # every rank ends with the full samples and coefficients
        same(r["s"], s_ref)
        same(r["f"], windowed)
        same(r["f2"], r["f"])
    assert np.abs(res[0]["f"] - flm).max() <= 1e-10


@pytest.mark.parametrize("L", [64, 256])
def test_processes_factors(tmp_path, L, grid_of):
    res = _run_ranks(tmp_path, L, "factors")
    g = grid_of(L)
    for r in res:
        flm = r["flm"]  # this rank's own two maps
        s_ref = osp.inverse_sht_batch(flm, g)
        same(r["s"], s_ref)
        same(r["f"], osp.forward_sht_batch(s_ref, g))
        same(r["f2"], r["f"])
