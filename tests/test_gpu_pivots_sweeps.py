"""GPU: in-house pivot discovery, every sweep variant under parity, device Legendre range KATs.

* The grid's pivot order (pivots.cu, hand-written: a partial-pivoting panel
  search in front of every breadth-first step) against LAPACK getrf's row
  order for the same blocks (scipy.linalg.lu_factor on the oracle's blocks,
  the reference's own block construction blocks.py:59-72).
* Each order-peeling sweep (persistent / GEMM / large / windowed) forced or
  selected by shape, with the variant that actually ran read back from the
  library (osph_last_sweep_kind), against the reference fixtures.
* osph_legendre_block at L=4096 on the reference's range KATs
  (pkg/tests/test_legendre.py:125-139): no overflow near the pole, populated
  away from it, an exact zero in the underflow region.
"""

import math

import numpy as np
import pytest

import paper_1403_4661_b200 as osp

pytestmark = pytest.mark.gpu


def tol_fwd(oracle_rt_err):
    return max(1e-11, 10.0 * oracle_rt_err)


def lapack_perm(a):
    """Row order of LU with partial pivoting (LAPACK dgetrf via scipy): perm[i] = row at position i."""
    from scipy.linalg import lu_factor

    _, piv = lu_factor(a, check_finite=False)
    perm = np.arange(a.shape[0])
    for i, j in enumerate(piv):
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def order_perm(perm_packed, L, m):
    off = m * L - m * (m - 1) // 2
    return perm_packed[off:off + L - m]


def swaps_needed(a, perm):
    """Interchanges LAPACK still makes on the rows in our order (0 = a partial-pivoting order)."""
    from scipy.linalg import lu_factor

    _, piv = lu_factor(a[perm], check_finite=False)
    return int(np.count_nonzero(piv != np.arange(a.shape[0])))


@pytest.mark.parametrize("L,ordering", [(64, "condmin"), (256, "condmin"), (256, "interleaved")])
def test_pivot_order_matches_lapack_getrf(L, ordering, grid_of):
    from oracle import optisph_oracle as O

    g = grid_of(L, ordering)
    plan = osp.transform.Plan(g.thetas, 1, 0)
    perm, _ = plan.pivots()
    plan.close()
    equal = 0
    orders = range(L) if L <= 64 else list(range(0, L, 5)) + [L - 1]
    for m in orders:
        mine = order_perm(perm, L, m)
        assert np.array_equal(np.sort(mine), np.arange(L - m)), m  # a permutation
        a = O.block(m, g.thetas)
        ref = lapack_perm(a)
        if np.array_equal(mine, ref):
            equal += 1
        elif ordering == "condmin":
            # a rounding-level near-tie may flip one choice; the order must still be a
            # partial-pivoting order of the block
            assert swaps_needed(a, mine) <= 2, m
    # condmin blocks are well conditioned: getrf's order exactly, order by order
    if ordering == "condmin":
        assert equal >= len(orders) - 2, f"{equal}/{len(orders)} orders equal"


@pytest.mark.parametrize("L,orders", [(2048, [0, 1, 700, 2040]), (4096, [0, 1000, 3000, 4090])])
def test_pivot_order_large_blocks(L, orders, grid_of, monkeypatch, fresh_gpu):
    """n up to 2048 (resident factor storage) and 4096 (windowed, 16-CTA clusters): our order
    is a partial-pivoting order of each block."""
    from oracle import optisph_oracle as O

    g = grid_of(L)
    monkeypatch.setenv("OSPH_PIVOTS_NOCACHE", "1")
    plan = osp.transform.Plan(g.thetas, 1, 0)
    perm, secs = plan.pivots()
    plan.close()
    print(f"L={L} pivot discovery {secs:.2f} s")
    for m in orders:
        mine = order_perm(perm, L, m)
        assert np.array_equal(np.sort(mine), np.arange(L - m)), m
        a = O.block(m, g.thetas)
        frac_equal = float(np.mean(mine == lapack_perm(a)))
        sw = swaps_needed(a, mine)
        print(f"  m={m}: {frac_equal:.4f} of positions equal getrf's, {sw} LAPACK swaps on our order")
        assert sw <= max(2, (L - m) // 200), m


def test_pivot_discovery_windowed_equals_resident(grid_of, monkeypatch):
    """Discovery window by window (factor storage in windows, window.cu) gives the same order."""
    g = grid_of(256)
    p1 = osp.transform.Plan(g.thetas, 1, 0)
    a, _ = p1.pivots()
    p1.close()
    monkeypatch.setenv("OSPH_PIVOTS_NOCACHE", "1")
    monkeypatch.setenv("OSPH_WINDOW_GB", "0.03")
    p2 = osp.transform.Plan(g.thetas, 1, 0)
    b, secs = p2.pivots()
    p2.close()
    assert secs > 0.0
    assert np.array_equal(a, b)


def test_pivot_order_cached_per_grid(grid_of):
    g = grid_of(256)
    p1 = osp.transform.Plan(g.thetas, 1, 0)
    a, _ = p1.pivots()
    p2 = osp.transform.Plan(g.thetas, 2, 0)
    b, secs = p2.pivots()
    p1.close()
    p2.close()
    assert np.array_equal(a, b)
    assert secs == 0.0  # second plan on the same grid: uploaded from the per-grid cache


# ---------------------------------------------------------------------------
# sweep variants


def _fresh_forward(grid, samples, real=False, env=None, monkeypatch=None):
    """Forward on a fresh plan (sweep configuration is chosen per plan); returns (flm, sweep kind)."""
    from paper_1403_4661_b200 import _lib

    if env:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
    B = samples.shape[0]
    plan = osp.transform.Plan(grid.thetas, B, 0)
    out = np.empty_like(samples)
    kind = _lib.OSPH_HOST | (_lib.OSPH_REAL if real else 0)
    plan.forward_raw(B, samples.ctypes.data, out.ctypes.data, kind, True)
    sweep = plan.last_sweep_kind()
    plan.close()
    if env:
        for k in env:
            monkeypatch.delenv(k)
    return out, sweep


@pytest.mark.parametrize("env,want", [({}, "blocked"), ({"OSPH_SWEEP_BLOCKED": "0"}, "persistent"),
                                      ({"OSPH_SWEEP_LARGE": "1"}, "large"),
                                      ({"OSPH_WINDOW_GB": "0.03"}, "windowed"),
                                      ({"OSPH_SB_SMALL": "0"}, "blocked")])
def test_sweep_variants_L256_reference(env, want, golden, grid_of, monkeypatch):
    """Config 2's grid and recipe through each sweep the library has, against the reference."""
    d = golden("ref_L256.npz")
    g = grid_of(256)
    samples = np.stack([d["cmb_samples"], d["white_samples"], d["real_samples"]])
    f, kind = _fresh_forward(g, samples, env=env, monkeypatch=monkeypatch)
    assert kind == want
    for i, recipe in enumerate(("cmb", "white", "real")):
        rt = np.abs(d[f"{recipe}_fwd"] - d[f"{recipe}_flm"]).max()
        assert np.abs(f[i] - d[f"{recipe}_fwd"]).max() <= tol_fwd(rt), recipe
        assert np.abs(f[i] - d[f"{recipe}_flm"]).max() <= tol_fwd(rt), recipe


@pytest.mark.parametrize("env,want", [({}, "blocked"), ({"OSPH_SWEEP_BLOCKED": "0"}, "persistent")])
def test_sweep_variants_bitwise_deterministic(env, want, grid_of, monkeypatch):
    """Config 2's shape (L=256, B=64): ten forward calls give the same bits (no racing reductions),
    for the blocked sweep (the default for batches) and the persistent one."""
    import torch

    from paper_1403_4661_b200 import _lib

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = grid_of(256)
    rng = np.random.default_rng(3)
    B = 64
    x = torch.from_numpy(rng.standard_normal((B, 256 * 256)) + 1j * rng.standard_normal((B, 256 * 256))).cuda()
    plan = osp.transform.Plan(g.thetas, B, 0)  # a fresh plan: the sweep is chosen per plan
    out = [torch.empty_like(x) for _ in range(2)]
    kind = _lib.OSPH_DEVICE
    plan.forward_raw(B, x.data_ptr(), out[0].data_ptr(), kind, False)
    assert plan.last_sweep_kind() == want
    for _ in range(9):
        plan.forward_raw(B, x.data_ptr(), out[1].data_ptr(), kind, False)
        assert torch.equal(out[1], out[0])
    fw = out[0].clone()
    plan.inverse_raw(B, x.data_ptr(), out[0].data_ptr(), kind)  # the inverse too (short rings fold without atomics)
    for _ in range(4):
        plan.inverse_raw(B, x.data_ptr(), out[1].data_ptr(), kind)
        assert torch.equal(out[1], out[0])
    plan.close()
    if want == "persistent":  # both sweeps solve the same systems: agreement far inside the parity tolerance
        monkeypatch.delenv("OSPH_SWEEP_BLOCKED")
        plan2 = osp.transform.Plan(g.thetas, B, 0)
        plan2.forward_raw(B, x.data_ptr(), out[1].data_ptr(), kind, False)
        assert plan2.last_sweep_kind() == "blocked"
        plan2.close()
        assert (out[1] - fw).abs().max().item() <= 1e-11 * max(1.0, fw.abs().max().item())


@pytest.mark.parametrize("env,want", [({}, "blocked"), ({"OSPH_SWEEP_BLOCKED": "0"}, "gemm")])
def test_config3_shape_gemm_sweep(env, want, golden, grid_of, monkeypatch):
    """BASELINE configs[2]: 256 real maps at L=512 (128 paired transforms) -> the blocked sweep
    (batched GEMM launches per block of orders; default) and the per-order GEMM sweep.

    Map 0 is the reference's own L=512 real-recipe map (fixture); every map's
    round trip and a sample of maps against the reference/oracle."""
    from oracle import optisph_oracle as O

    d = golden("ref_L512.npz")
    g = grid_of(512)
    L, B = 512, 256
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(31)
    flm = np.empty((B, L * L), dtype=np.complex128)
    flm[0] = d["flm"]
    for b in range(1, B):
        flm[b] = O.config_coefficients(L, rng, spectrum="cmb", real=True)
    plan = osp.transform.Plan(g.thetas, B, 0)
    from paper_1403_4661_b200 import _lib

    s = np.empty_like(flm)
    plan.inverse_raw(B, flm.ctypes.data, s.ctypes.data, _lib.OSPH_HOST | _lib.OSPH_REAL)
    assert np.abs(s[0] - d["samples"]).max() <= 1e-12 * max(1.0, np.abs(d["samples"]).max())
    f = np.empty_like(flm)
    plan.forward_raw(B, s.ctypes.data, f.ctypes.data, _lib.OSPH_HOST | _lib.OSPH_REAL, True)
    assert plan.last_sweep_kind() == want
    plan.close()
    rt = np.abs(d["fwd"] - d["flm"]).max()
    assert np.abs(f[0] - d["fwd"]).max() <= tol_fwd(rt)
    assert np.abs(f - flm).max() <= tol_fwd(rt)
    # oracle (the reference's algorithm in C + LAPACK) on a sample of the other maps
    for b in (1, 77, 255):
        ref_s = O.inverse_sht(flm[b], g.thetas)
        assert np.abs(s[b] - ref_s.real).max() <= 1e-12 * max(1.0, np.abs(ref_s).max())


def test_config3_shape_without_gemm_sweep(grid_of, monkeypatch):
    """Same shape class with the GEMM sweep disabled: persistent teams in waves."""
    from oracle import optisph_oracle as O

    g = grid_of(512)
    L, B = 512, 96
    rng = np.random.default_rng(32)
    flm = np.stack([O.config_coefficients(L, rng, spectrum="cmb", real=True) for _ in range(B)])
    s = osp.inverse_sht_batch(flm, g, real=True)
    ref, kind0 = _fresh_forward(g, s, real=True)
    f, kind = _fresh_forward(g, s, real=True, env={"OSPH_SWEEP_NO_GEMM": "1"}, monkeypatch=monkeypatch)
    assert kind0 == "blocked" and kind == "persistent"
    assert np.abs(f - flm).max() <= 1e-11
    assert np.abs(f - ref).max() <= 1e-12


# ---------------------------------------------------------------------------
# device Legendre rows at L=4096: the reference's rescaling-range KATs


def test_legendre_block_range_L4096(fresh_gpu):
    import ctypes

    import torch

    from oracle import optisph_oracle as O
    from paper_1403_4661_b200 import _lib, sampling

    L = 4096
    th = sampling.equiangular_candidates(L).copy()
    th[1] = math.pi / 2  # the reference's "away from the pole" column (test_legendre.py:131)
    assert th[0] == math.pi / (2 * L - 1)
    plan = osp.transform.Plan(th, 1, 0)
    for m in (0, 1, 100, 1000, 2000, 2500, 4095):
        buf = torch.empty((L - m, L), dtype=torch.float64, device="cuda")
        _lib.raise_for(plan._lib.osph_legendre_block(plan.handle, m, ctypes.c_void_p(buf.data_ptr()), L,
                                                     _lib.OSPH_DEVICE))
        got = buf.T.cpu().numpy()  # (rings, degrees)
        assert np.all(np.isfinite(got)), m
        ref = O.legendre_table(m, th, L)
        # fma recurrence vs the reference's plain one, up to 4096 steps deep: measured 4.3e-12 (m=0)
        # and 1.2e-11 (m=1) of the largest value
        assert np.abs(got - ref).max() <= 5e-11 * np.abs(ref).max(), m
        if m == 2000:
            assert np.abs(got[1]).max() > 1e-3  # populated, not flushed
        if m == 4095:
            assert got[0, 0] == 0.0  # sin(theta)^4095 underflows: exact zero
    plan.close()
