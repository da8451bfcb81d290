"""CPU: the spin-weighted path's oracle pinned to the reference, and the
C-ABI seed constants (osph_spin_seed, host-only) against the exact rationals.

Fixtures: tests/golden/ref_spin.npz (tests/golden/make_golden_spin.py, run
against the reference in the build container)."""

import ctypes
import math

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import optisph_oracle as O


@pytest.fixture(scope="module")
def ref():
    return np.load(GOLDEN / "ref_spin.npz")


def test_oracle_spin_tables_match_reference(ref):
    n = 0
    for key in ref.files:
        if key.startswith("tab_"):
            _, L, s, m = key.split("_")
            L, s, m = int(L[1:]), int(s[1:]), int(m[1:])
            assert np.array_equal(O.spin_table(s, m, ref[f"L{L}_thetas"], L), ref[key]), key
            n += 1
    assert n > 50


@pytest.mark.parametrize("L", [16, 32, 64])
@pytest.mark.parametrize("s", [1, -1, 2, 3])
def test_oracle_spin_transforms_match_reference(ref, L, s):
    th = ref[f"L{L}_thetas"]
    flm = ref[f"L{L}_s{s}_flm"]
    assert np.array_equal(O.spin_inverse_sht(flm, th, s), ref[f"L{L}_s{s}_samples"])
    assert np.array_equal(O.spin_forward_sht(ref[f"L{L}_s{s}_samples"], th, s), ref[f"L{L}_s{s}_fwd"])


@pytest.mark.parametrize("s", [1, 2, -3])
def test_oracle_spin_least_squares_noise(ref, s):
    """Inconsistent (not band-limited) samples: the tall blocks' least-squares answers."""
    th = ref["L16_thetas"]
    assert np.array_equal(O.spin_forward_sht(ref[f"L16_s{s}_noise"], th, s), ref[f"L16_s{s}_noise_fwd"])


def test_oracle_spin_table_against_wigner_sum():
    """legendre.py's spin columns against the explicit Wigner-d sum (test_legendre.py:193-204)."""
    worst = 0.0
    for s in (-2, -1, 1, 2):
        for m in range(-3, 4):
            for theta in (0.2, 1.1, 2.5):
                col = O.spin_table(s, m, [theta], 4)[0]
                lo = max(abs(m), abs(s))
                for j, ell in enumerate(range(lo, 4)):
                    worst = max(worst, abs(col[j] - O.spin_direct(s, ell, m, theta)))
    assert worst <= 1e-12


def test_oracle_spin_zero_table_is_scalar():
    th = np.linspace(0.1, 3.0, 7)
    for m in (-4, -1, 0, 2, 5):
        assert np.abs(O.spin_table(0, m, th, 12) - O.legendre_table(m, th, 12)).max() <= 1e-12


def _seed(lib, s, m):
    out = [ctypes.c_int(), ctypes.c_double(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()]
    assert lib.osph_spin_seed(s, m, *[ctypes.byref(v) for v in out]) == 0
    return tuple(v.value for v in out)


def test_capi_spin_seed_matches_exact_rationals():
    """osph_spin_seed (prime-exponent products in long double) == Fraction arithmetic, bit for bit."""
    from paper_1403_4661_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(3)
    cases = [(s, m) for s in (-3, -1, 1, 2, 5) for m in range(-12, 13)]
    cases += [(int(s), int(m)) for s, m in zip(rng.integers(-4095, 4096, 120), rng.integers(-4095, 4096, 120))]
    cases += [(1, 4095), (-1, -4095), (4095, 0), (-4095, 4095), (2, 2048), (-7, -3000)]
    for s, m in cases:
        assert _seed(lib, s, m) == O.spin_seed_constants(s, m), (s, m)


def test_capi_spin_seed_reproduces_reference_seed_state(ref):
    """The reference's _spin_seed (mantissa, offset) at three co-latitudes, rebuilt
    from the C constants with the reference's multiply/rescale loop."""
    from paper_1403_4661_b200 import _lib

    lib = _lib.load()
    th = ref["seed_thetas"]
    ch, sh = np.cos(th / 2.0), np.sin(th / 2.0)
    for (s, m), mant_ref, off_ref in zip(ref["seed_rows"], ref["seed_mant"], ref["seed_off"]):
        j, scale, off0, es, ec = _seed(lib, int(s), int(m))
        for i in range(th.size):
            mant, off = scale, off0
            for _ in range(es):
                mant *= sh[i]
                if abs(mant) < 2.0**-500 and mant != 0.0:
                    mant *= 2.0**1000
                    off -= 1000
            for _ in range(ec):
                mant *= ch[i]
                if abs(mant) < 2.0**-500 and mant != 0.0:
                    mant *= 2.0**1000
                    off -= 1000
            assert mant == mant_ref[i] and off == off_ref[i], (s, m, i)
