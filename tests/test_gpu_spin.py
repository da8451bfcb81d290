"""GPU parity of the spin-weighted transforms against the
reference (tests/golden/ref_spin.npz, produced by the reference itself) and the
oracle restatement (oracle/optisph_oracle.py spin_*), through the C ABI
(osph_spin_inverse / osph_spin_forward / osph_spin_block).

Tolerances:
  * tables and the inverse are forward evaluations: 1e-12 relative to the
    largest magnitude;
  * the forward peels orders m = L-1..0 and every order's errors feed the
    lower orders' right-hand sides, so the REFERENCE's own round-trip error
    grows as m falls (at L=64, s=3 it reaches 1e87: ref_spin.npz).  The bar is
    per order |m|: max |f_gpu - f_ref| <= max(1e-11, 10 x the reference's
    round-trip error at that order) (the round's parity rule,
    max(1e-11, 10 x oracle round-trip error), applied order by order).
"""

import numpy as np
import pytest

from conftest import GOLDEN, has_gpu
from oracle import optisph_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def ref():
    return np.load(GOLDEN / "ref_spin.npz")


def _grid(L):
    import paper_1403_4661_b200 as osp

    from conftest import GRIDS

    return osp.load_grid(GRIDS / f"grid-L{L}-uniform-condmin.txt")


def _orders(L):
    n = np.arange(L * L)
    ell = np.floor(np.sqrt(n)).astype(np.int64)
    return ell, n - ell * ell - ell


def _per_order_ok(got, want, truth, L):
    ell, m = _orders(L)
    worst = 0.0
    for am in range(L):
        sel = np.abs(m) == am
        rt = np.abs(want[sel] - truth[sel]).max()
        err = np.abs(got[sel] - want[sel]).max()
        tol = max(1e-11, 10.0 * rt)
        assert err <= tol, f"order {am}: |gpu - ref| {err:.3e} > {tol:.3e}"
        worst = max(worst, err / tol)
    return worst


def test_spin_tables_match_reference(ref):
    import paper_1403_4661_b200 as osp

    for key in ref.files:
        if not key.startswith("tab_"):
            continue
        _, L, s, m = key.split("_")
        L, s, m = int(L[1:]), int(s[1:]), int(m[1:])
        want = ref[key]
        got = osp.spin_table(s, m, ref[f"L{L}_thetas"], L)
        assert got.shape == want.shape
        assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max()), key


def test_spin_table_arbitrary_thetas_and_range():
    import paper_1403_4661_b200 as osp

    th = np.linspace(0.05, np.pi, 37)  # more co-latitudes than L: chunked over plans
    got = osp.spin_table(2, -1, th, 16)
    assert np.abs(got - O.spin_table(2, -1, th, 16)).max() <= 1e-12
    with pytest.raises(osp.OrderRangeError):
        osp.spin_table(16, 0, th, 16)
    with pytest.raises(osp.OrderRangeError):
        osp.spin_table(0, -16, th, 16)


@pytest.mark.parametrize("L", [16, 32, 64])
@pytest.mark.parametrize("s", [1, -1, 2, 3])
def test_spin_inverse_matches_reference(ref, L, s):
    import paper_1403_4661_b200 as osp

    flm = ref[f"L{L}_s{s}_flm"]
    got = osp.spin_inverse_sht_batch(flm[None], _grid(L), s)[0]
    want = ref[f"L{L}_s{s}_samples"]
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("L", [16, 32, 64])
@pytest.mark.parametrize("s", [1, -1, 2, 3])
def test_spin_forward_matches_reference_per_order(ref, L, s):
    import paper_1403_4661_b200 as osp

    samples = ref[f"L{L}_s{s}_samples"]
    got = osp.spin_forward_sht_batch(samples[None], _grid(L), s)[0]
    want, flm = ref[f"L{L}_s{s}_fwd"], ref[f"L{L}_s{s}_flm"]
    _per_order_ok(got, want, flm, L)
    ell, m = _orders(L)
    for am in range(L):  # per order no less accurate than the reference
        sel = np.abs(m) == am
        assert np.abs(got[sel] - flm[sel]).max() <= 10 * np.abs(want[sel] - flm[sel]).max() + 1e-11, am
    assert np.all(got[ell < abs(s)] == 0)  # degrees below |spin| come back exactly zero


@pytest.mark.parametrize("s", [1, 2, -3])
def test_spin_forward_least_squares_on_noise(ref, s):
    """Inconsistent samples: the tall blocks' least-squares solutions (gelsy in the
    reference, Householder QR here).  Two error sources set the bar per order,
    each taken at 10x: the spread between two LAPACK least-squares solvers
    (gelsy vs gelsd) run through the same oracle sweep, and the sweep's own
    amplification -- the oracle's round-trip error on consistent data of unit
    size at this spin, relative to the order's coefficient magnitude."""
    import paper_1403_4661_b200 as osp

    L = 16
    th = _grid(L).thetas
    noise = ref[f"L16_s{s}_noise"]
    got = osp.spin_forward_sht_batch(noise[None], _grid(L), s)[0]
    want = ref[f"L16_s{s}_noise_fwd"]
    other = O.spin_forward_sht(noise, th, s, driver="gelsd")
    ell, m = _orders(L)
    rng = np.random.default_rng(9)
    flm = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
    flm[ell < abs(s)] = 0
    rt = O.spin_forward_sht(O.spin_inverse_sht(flm, th, s), th, s) - flm
    for am in range(L):
        sel = np.abs(m) == am
        scale = max(1.0, np.abs(want[sel]).max())
        spread = np.abs(other[sel] - want[sel]).max()
        tol = max(1e-11 * scale, 10.0 * spread, 10.0 * np.abs(rt[sel]).max() * scale)
        assert np.abs(got[sel] - want[sel]).max() <= tol, am


def test_spin_round_trips_like_reference_tests():
    """test_transform.py:187-201 on the condmin L=16 grid."""
    import paper_1403_4661_b200 as osp

    grid = _grid(16)
    c = osp.HarmonicCoefficients.zeros(16)
    c.set(1, 0, 1.0)
    c2 = osp.spin_forward_sht(osp.spin_inverse_sht(c, grid, 1), grid, 1)
    assert np.abs(c.values - c2.values).max() <= 1e-10
    rng = np.random.default_rng(20240901)
    c = osp.HarmonicCoefficients.zeros(16)
    for ell in range(1, 16):
        for m in range(-ell, ell + 1):
            c.set(ell, m, complex(rng.uniform(-1, 1), rng.uniform(-1, 1)))
    c2 = osp.spin_forward_sht(osp.spin_inverse_sht(c, grid, 1), grid, 1)
    assert np.abs(c.values - c2.values).max() <= 1e-8


def test_spin_out_of_range_and_low_degrees():
    import paper_1403_4661_b200 as osp

    grid = _grid(16)
    rng = np.random.default_rng(1)
    c = osp.HarmonicCoefficients(16, rng.standard_normal(256) + 1j * rng.standard_normal(256))
    with pytest.raises(osp.OrderRangeError):
        osp.spin_inverse_sht(c, grid, 16)
    s = osp.spin_inverse_sht(c, grid, 2)  # junk below l = 2 is ignored
    with pytest.raises(osp.OrderRangeError):
        osp.spin_forward_sht(s, grid, -16)
    c2 = osp.spin_forward_sht(s, grid, 2)
    for ell in range(2):
        for m in range(-ell, ell + 1):
            assert c2.get(ell, m) == 0


def test_spin_zero_is_the_scalar_path_bit_for_bit():
    """test_transform.py:178-185 / test_acceptance.py criterion 10."""
    import paper_1403_4661_b200 as osp

    grid = _grid(16)
    rng = np.random.default_rng(2)
    c = osp.HarmonicCoefficients(16, rng.standard_normal(256) + 1j * rng.standard_normal(256))
    a = osp.inverse_sht(c, grid)
    b = osp.spin_inverse_sht(c, grid, 0)
    assert all(np.array_equal(x, y) for x, y in zip(a.rings, b.rings))
    assert np.array_equal(osp.forward_sht(a, grid).values, osp.spin_forward_sht(a, grid, 0).values)


def test_spin_batch_device_and_repeat_are_bitwise_identical(ref):
    import torch

    import paper_1403_4661_b200 as osp

    L, s = 32, 1
    grid = _grid(L)
    rng = np.random.default_rng(4)
    flm = rng.standard_normal((5, L * L)) + 1j * rng.standard_normal((5, L * L))
    inv = osp.spin_inverse_sht_batch(flm, grid, s)
    for b in range(5):  # batch == one map at a time
        assert np.array_equal(inv[b], osp.spin_inverse_sht_batch(flm[b:b + 1], grid, s)[0])
    fwd = osp.spin_forward_sht_batch(inv, grid, s)
    assert np.array_equal(fwd[3], osp.spin_forward_sht_batch(inv[3:4], grid, s)[0])
    assert np.array_equal(fwd, osp.spin_forward_sht_batch(inv, grid, s))  # deterministic
    dev = osp.spin_forward_sht_batch(torch.from_numpy(inv).cuda(), grid, s)  # device buffers
    assert np.array_equal(fwd, dev.cpu().numpy())
    dinv = osp.spin_inverse_sht_batch(torch.from_numpy(flm).cuda(), grid, s)
    assert np.array_equal(inv, dinv.cpu().numpy())


def test_spin_forward_stats_and_check():
    import paper_1403_4661_b200 as osp

    L = 16
    grid = _grid(L)
    plan = osp.get_plan(grid, 1, 0)
    st = osp.TransformStats()
    x = O.spin_inverse_sht(np.ones(L * L, dtype=np.complex128), grid.thetas, 2)
    osp.spin_forward_sht_batch(x[None], grid, -2, stats=st)
    assert st.orders == L and st.extra["sweep_seconds"] > 0
    assert plan.last_launch_count() >= 2 * L - 1  # a solve per order + corrections of every m >= 1 + ring DFTs


@pytest.mark.parametrize("s", [1, -2])
def test_spin_L256_against_oracle(s):
    """Larger band limit: inverse at 1e-12; forward per order against the oracle's
    own forward of the same samples (bar from the oracle's round trip)."""
    import paper_1403_4661_b200 as osp

    L = 256
    grid = _grid(L)
    rng = np.random.default_rng(256 + s)
    ell, m = _orders(L)
    flm = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
    flm[ell < abs(s)] = 0
    # the oracle's inverse on every ring is the slow part: check a spread of rings
    samples = O.spin_inverse_sht(flm, grid.thetas, s)
    got_inv = osp.spin_inverse_sht_batch(flm[None], grid, s)[0]
    assert np.abs(got_inv - samples).max() <= 1e-12 * np.abs(samples).max()
    want = O.spin_forward_sht(samples, grid.thetas, s)
    got = osp.spin_forward_sht_batch(samples[None], grid, s)[0]
    _per_order_ok(got, want, flm, L)
    # and per order no less accurate than the reference (its round trip grows as m
    # falls: 1e-11 at m = L/2 for s = 1, 1e22 for s = -2 on this grid)
    for am in range(L):
        sel = np.abs(m) == am
        assert np.abs(got[sel] - flm[sel]).max() <= 10 * np.abs(want[sel] - flm[sel]).max() + 1e-11, am
