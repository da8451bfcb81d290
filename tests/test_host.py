"""CPU: host-side logic of the package and the C-ABI boundary (no GPU compute)."""

import ctypes
import re
import zlib
from pathlib import Path

import numpy as np
import pytest

import paper_1403_4661_b200 as osp
from paper_1403_4661_b200 import _lib
from conftest import GRIDS, ROOT, has_gpu


def test_index_bijection():
    L = 9
    seen = {osp.HarmonicCoefficients.index(l, m) for l in range(L) for m in range(-l, l + 1)}
    assert seen == set(range(L * L))


def test_order_slice_round_trip(rng):
    L = 7
    c = osp.HarmonicCoefficients(L, rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L))
    for m in range(-(L - 1), L):
        assert np.array_equal(c.order_slice(m), [c.get(l, m) for l in range(abs(m), L)])
    d = osp.HarmonicCoefficients.zeros(L)
    for m in range(-(L - 1), L):
        d.set_order_slice(m, c.order_slice(m))
    assert np.array_equal(c.values, d.values)


def test_samples_layout(rng):
    L = 6
    flat = rng.standard_normal(L * L) + 0j
    s = osp.SpatialSamples.from_flat(L, flat)
    assert [len(r) for r in s.rings] == [2 * k + 1 for k in range(L)]
    assert np.array_equal(s.flatten(), flat)
    assert s.sample_count == L * L
    with pytest.raises(osp.BandLimitError):
        osp.SpatialSamples.from_flat(L, flat[:-1])


@pytest.mark.parametrize("L", [8, 16, 32, 64, 256])
def test_grid_files_load_and_round_trip(L, tmp_path):
    g = osp.load_grid(GRIDS / f"grid-L{L}-uniform-condmin.txt")
    assert g.band_limit == L and g.ordering is osp.Ordering.CONDITION_MINIMIZED
    np.testing.assert_array_equal(g.thetas, osp.equiangular_candidates(L)[g.permutation])
    out = tmp_path / "g.txt"
    osp.save_grid(g, out)
    assert out.read_text() == (GRIDS / f"grid-L{L}-uniform-condmin.txt").read_text()


def test_interleaved_matches_reference_file():
    for L in (16, 64, 256):
        ref = osp.load_grid(GRIDS / f"grid-L{L}-uniform-interleaved.txt")
        mine = osp.interleaved_grid(L)
        assert np.array_equal(ref.permutation, mine.permutation)
        assert np.array_equal(ref.thetas, mine.thetas)


def test_grid_crc_and_format_errors(tmp_path):
    src = (GRIDS / "grid-L16-uniform-condmin.txt").read_text().splitlines()
    bad = tmp_path / "bad.txt"
    bad.write_text("\n".join(src[:-1] + ["crc32 00000000"]) + "\n")
    with pytest.raises(osp.FileFormatError):
        osp.load_grid(bad)
    bad.write_text("nonsense\n")
    with pytest.raises(osp.FileFormatError):
        osp.load_grid(bad)
    payload = "\n".join(src[:4] + src[5:-1]) + "\n"  # one permutation line missing
    bad.write_text(payload + f"crc32 {zlib.crc32(payload.encode()):08x}\n")
    with pytest.raises(osp.FileFormatError):
        osp.load_grid(bad)


def test_grid_invariants():
    with pytest.raises(ValueError):
        osp.ColatitudeGrid(3, np.array([0.5, 0.5, 1.0]), np.array([0, 1, 2]))
    with pytest.raises(ValueError):
        osp.ColatitudeGrid(2, np.array([0.5, 1.0]), np.array([0, 0]))


def _declared_symbols():
    text = (ROOT / "include" / "osph.h").read_text()
    return sorted(set(re.findall(r"\b(osph_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    declared = _declared_symbols()
    assert "osph_forward" in declared and "osph_inverse" in declared
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), "ctypes binding and header disagree"
    assert lib.osph_abi_version() == _lib.ABI_VERSION


def test_error_codes_and_messages_without_compute():
    lib = _lib.load()
    # argument validation happens before any device work
    h = ctypes.c_void_p()
    th = np.linspace(0.1, 3.0, 8)
    dev = (ctypes.c_int * 1)(0)
    assert lib.osph_plan_create(8, th.ctypes.data_as(ctypes.c_void_p), 1, 0, ctypes.cast(dev, ctypes.c_void_p),
                                ctypes.byref(h)) == _lib.OSPH_ERR_ARG  # ndev must be >= 1
    assert lib.osph_plan_create(0, th.ctypes.data_as(ctypes.c_void_p), 1, 1, ctypes.cast(dev, ctypes.c_void_p), ctypes.byref(h)) == _lib.OSPH_ERR_ARG
    assert "band limit" in _lib.last_error()
    bad = th.copy()
    bad[3] = -1.0
    assert lib.osph_plan_create(8, bad.ctypes.data_as(ctypes.c_void_p), 1, 1, ctypes.cast(dev, ctypes.c_void_p), ctypes.byref(h)) == _lib.OSPH_ERR_ARG
    assert lib.osph_inverse(None, 1, None, None, 0) == _lib.OSPH_ERR_ARG
    # shard partition (pure host logic): blocks descend with the rank and tile [0, L)
    for L, n, mode in ((64, 2, _lib.SHARD_CHAIN), (256, 8, _lib.SHARD_FACTORS), (8, 8, _lib.SHARD_CHAIN)):
        prev_lo, k_prev = L, 0
        for r in range(n):
            v = [ctypes.c_int() for _ in range(4)]
            assert lib.osph_shard_range(L, r, n, mode, *[ctypes.byref(x) for x in v]) == _lib.OSPH_OK
            m_lo, m_hi, k_lo, k_hi = (x.value for x in v)
            assert m_hi == prev_lo - 1 and m_lo <= m_hi
            prev_lo = m_lo
            if mode == _lib.SHARD_CHAIN:
                assert k_lo == k_prev and k_hi > k_lo
                k_prev = k_hi
        assert prev_lo == 0 and (mode != _lib.SHARD_CHAIN or k_prev == L)
    v = [ctypes.c_int() for _ in range(4)]
    assert lib.osph_shard_range(8, 0, 9, _lib.SHARD_CHAIN, *[ctypes.byref(x) for x in v]) == _lib.OSPH_ERR_ARG
    out = np.zeros(4)
    ring = np.zeros(4, dtype=complex)
    assert lib.osph_ring_analysis(ring.ctypes.data_as(ctypes.c_void_p), 4, 0,
                                  out.ctypes.data_as(ctypes.c_void_p), 0) == _lib.OSPH_ERR_ARG


@pytest.mark.skipif(has_gpu(), reason="checks the no-device path")
def test_no_cpu_fallback_without_gpu():
    """The product refuses to run without a CUDA device instead of falling back."""
    g = osp.load_grid(GRIDS / "grid-L8-uniform-condmin.txt")
    with pytest.raises(osp.DeviceError):
        osp.inverse_sht(osp.HarmonicCoefficients.zeros(8), g)
    with pytest.raises(osp.DeviceError):
        osp.forward_sht(osp.SpatialSamples.zeros(8), g)


def test_python_api_validation_before_device():
    g = osp.load_grid(GRIDS / "grid-L8-uniform-condmin.txt")
    with pytest.raises(osp.BandLimitError):
        osp.inverse_sht(osp.HarmonicCoefficients.zeros(4), g)
    with pytest.raises(ValueError):
        osp.forward_sht(osp.SpatialSamples.zeros(8), g, method="magic")
    with pytest.raises(osp.AliasingError):
        osp.ring_analysis(np.zeros(3, dtype=complex), 2)
    with pytest.raises(ValueError):
        osp.ring_analysis(np.zeros(4, dtype=complex), 0)
