"""GPU: the blocked order-peeling sweep (sweep_block.cu) and the register-resident ring DFTs
(fft_reg.cuh) at band limits and batch sizes around their block / class boundaries.

* The blocked sweep (blocks of 32 orders, in-block aliasing by the scalar recurrence) against
  the oracle's forward (the reference's `_forward_spectral` loop, transform.py:436-467) and
  against the persistent sweep, for L that are / are not multiples of 32, L <= 32 (the final
  block alone), batches that do not fill the 8-map GEMM tiles, and real (paired) maps.
* Every ring-DFT class: direct (n <= 63), register-resident 256 / 512 / 1024 / 2048, the
  shared-memory transform, against the oracle's inverse (numpy.fft per ring, transform.py:334-344)
  and with the register classes switched off (OSPH_RING_REG=0).
"""

import numpy as np
import pytest

import paper_1403_4661_b200 as osp

pytestmark = pytest.mark.gpu


def _grid(L, grid_of):
    from paper_1403_4661_b200 import gridopt

    try:
        return grid_of(L)
    except FileNotFoundError:
        return gridopt.make_grid(L, ordering=osp.Ordering.CONDITION_MINIMIZED)


def _forward(grid, samples, env, monkeypatch, real=False):
    from paper_1403_4661_b200 import _lib

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    B = samples.shape[0]
    plan = osp.transform.Plan(grid.thetas, B, 0)
    out = np.empty_like(samples)
    plan.forward_raw(B, samples.ctypes.data, out.ctypes.data, _lib.OSPH_HOST | (_lib.OSPH_REAL if real else 0), True)
    kind = plan.last_sweep_kind()
    plan.close()
    for k in env:
        monkeypatch.delenv(k)
    return out, kind


@pytest.mark.parametrize("L,B", [(8, 3), (32, 5), (33, 16), (64, 17), (100, 9), (127, 24), (160, 16), (200, 7)])
def test_blocked_sweep_vs_oracle_and_persistent(L, B, grid_of, monkeypatch):
    from oracle import optisph_oracle as O

    g = _grid(L, grid_of)
    rng = np.random.default_rng(1000 + L)
    flm = np.stack([O.config_coefficients(L, rng, spectrum="cmb", real=False) for _ in range(B)])
    s = osp.inverse_sht_batch(flm, g)
    fb, kb = _forward(g, s, {"OSPH_SWEEP_BLOCKED": "1"}, monkeypatch)
    fp, kp = _forward(g, s, {"OSPH_SWEEP_BLOCKED": "0"}, monkeypatch)
    assert kb == "blocked" and kp == "persistent"
    scale = max(1.0, np.abs(flm).max())
    for b in (0, B - 1):  # the reference's algorithm on the same samples
        ref = O.forward_sht(s[b], g.thetas, method="spectral")
        rt = np.abs(ref - flm[b]).max()
        assert np.abs(fb[b] - ref).max() <= max(1e-11, 10.0 * rt) * scale, (L, b)
    assert np.abs(fb - flm).max() <= 1e-10 * scale
    assert np.abs(fb - fp).max() <= 1e-11 * scale


def test_blocked_sweep_real_maps_and_odd_batch(grid_of, monkeypatch):
    """Real maps are paired into complex transforms (OSPH_REAL): 37 maps -> 19 pairs at L = 96."""
    from oracle import optisph_oracle as O

    L, B = 96, 37
    g = _grid(L, grid_of)
    rng = np.random.default_rng(77)
    flm = np.stack([O.config_coefficients(L, rng, spectrum="cmb", real=True) for _ in range(B)])
    s = osp.inverse_sht_batch(flm, g, real=True)
    f, kind = _forward(g, s, {}, monkeypatch, real=True)
    assert kind == "blocked"  # the default at L <= 512
    assert np.abs(f - flm).max() <= 1e-11
    ref = O.forward_sht(s[5], g.thetas, method="spectral")
    assert np.abs(f[5] - ref).max() <= 1e-11


def test_blocked_sweep_ill_conditioned_order_reported(grid_of, monkeypatch):
    """check=True through the blocked sweep reports the reference's failing order on the singular grid."""
    g = grid_of(256, "interleaved")
    rng = np.random.default_rng(5)
    B = 16
    s = rng.standard_normal((B, 256 * 256)) + 1j * rng.standard_normal((B, 256 * 256))
    with pytest.raises(osp.IllConditionedSolveError) as ei:
        osp.forward_sht_batch(s, g, check=True)
    assert ei.value.order == 220


@pytest.mark.parametrize("L", [40, 70, 140, 260, 300, 520])
def test_ring_classes_vs_oracle(L, grid_of, monkeypatch):
    """Rings of every DFT class at this L: direct, 256 / 512 / 1024 / 2048-point register-resident
    (fft sizes >= 2n-1), shared-memory above; inverse against the oracle, forward by round trip,
    and both against the shared-memory transforms alone (OSPH_RING_REG=0)."""
    from oracle import optisph_oracle as O

    g = _grid(L, grid_of)
    rng = np.random.default_rng(2000 + L)
    B = 5
    flm = np.stack([O.config_coefficients(L, rng, spectrum="cmb", real=False) for _ in range(B)])
    s = osp.inverse_sht_batch(flm, g)
    rings = sorted({0, 1, 31, 32, 63, 64, 127, 128, 255, 256, 299, 511, L - 1} & set(range(L)))
    ref = O.inverse_rings(flm[2], g.thetas, rings)
    for k in rings:
        r = ref[k]
        got = s[2, k * k:(k + 1) * (k + 1)]
        assert np.abs(got - r).max() <= 1e-12 * max(1.0, np.abs(r).max()), (L, k)
    f = osp.forward_sht_batch(s, g, check=False)
    tol = 1e-11 if L <= 300 else 1e-9  # the chain's own amplification at L = 520 (reference: same order)
    assert np.abs(f - flm).max() <= tol * max(1.0, np.abs(flm).max())
    monkeypatch.setenv("OSPH_RING_REG", "0")
    plan = osp.transform.Plan(g.thetas, B, 0)
    from paper_1403_4661_b200 import _lib

    s2 = np.empty_like(s)
    plan.inverse_raw(B, flm.ctypes.data, s2.ctypes.data, _lib.OSPH_HOST)
    plan.close()
    monkeypatch.delenv("OSPH_RING_REG")
    assert np.abs(s2 - s).max() <= 1e-12 * max(1.0, np.abs(s).max())
