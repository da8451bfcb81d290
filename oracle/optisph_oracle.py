"""CPU oracle for the forward/inverse SHT hot path -- TEST INFRASTRUCTURE ONLY.

This module restates the reference package ``optisph`` (read-only at
/root/reference/pkg/src/optisph) for the north_star path.  It is the checker
for the CUDA implementation: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline leg and ``--impl reference``) may import it.  The
product package ``paper_1403_4661_b200`` never imports it and has no CPU
fallback.

The scalar inner loops live in ``oracle_kernels.c`` (restating the reference's
numba kernels, see that file's header); the library calls the reference makes
(``numpy.fft``, ``scipy.linalg.lstsq(lapack_driver="gelsy")``,
``numpy.linalg.svd``) are made here exactly as the reference makes them.

Parity pin: ``tests/test_oracle.py`` checks every function below against
fixtures produced by running the reference itself in the build container
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import zlib
from functools import lru_cache
from pathlib import Path

import numpy as np
from scipy import linalg

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"

TWO_PI = 2.0 * np.pi  # blocks.py:24
FOUR_PI = 4.0 * math.pi  # legendre.py:26
SOLVE_RCOND = 1e-14  # blocks.py:27
GRID_MAGIC = "OPTISPH-GRID v1"  # sampling.py:32


class OracleIllConditioned(RuntimeError):
    """Mirror of optisph.errors.IllConditionedSolveError (errors.py:28-36)."""

    def __init__(self, order: int, kappa: float):
        super().__init__(
            f"order {order} system is numerically singular (condition number {kappa:.3e})"
        )
        self.order = order
        self.kappa = kappa


def build() -> Path:
    """Compile oracle_kernels.c with gcc (no-op when up to date)."""
    src = _HERE / "oracle_kernels.c"
    if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


_lib = None


def _clib():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        I = ctypes.c_int64
        D = ctypes.c_double
        lib.oracle_legendre_kernel.argtypes = [P, P, I, I, I, D, P, P, P, P]
        lib.oracle_g_accumulate.argtypes = [P, P, I, P, P, P, P, P, I, P]
        lib.oracle_fold_bins.argtypes = [P, P, I, P]
        lib.oracle_peel_analyze.argtypes = [P, P, I, I, P, P]
        lib.oracle_peel_update.argtypes = [P, P, I, I, P, P]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# grids (sampling.py)


def equiangular_candidates(L: int) -> np.ndarray:
    """pi*(2t+1)/(2L-1), t = 0..L-1 (sampling.py:97-105)."""
    t = np.arange(L)
    return np.pi * ((2 * t + 1) / (2 * L - 1))


def interleaved_permutation(L: int) -> np.ndarray:
    """Default ring assignment (sampling.py:181-189)."""
    perm = np.empty(L, dtype=np.int64)
    perm[0] = L - 1
    for k in range(1, L):
        perm[k] = (k - 1) // 2 if k % 2 else L - 1 - k // 2
    return perm


def load_grid_file(path) -> tuple[int, np.ndarray, np.ndarray]:
    """Parse an OPTISPH-GRID v1 file (sampling.py:334-370) -> (L, perm, thetas).

    Only the uniform measure is supported here (the hot-path grids).
    """
    text = Path(path).read_text(encoding="ascii")
    lines = text.splitlines()
    if not lines or lines[0] != GRID_MAGIC:
        raise ValueError(f"{path}: bad grid header")
    payload = "\n".join(lines[:-1]) + "\n"
    if zlib.crc32(payload.encode("ascii")) != int(lines[-1].split()[1], 16):
        raise ValueError(f"{path}: crc mismatch")
    L = int(lines[1].split()[1])
    if lines[2].split()[1] != "uniform":
        raise ValueError("oracle supports uniform-measure grids only")
    perm = np.array([int(s) for s in lines[4:-1]], dtype=np.int64)
    return L, perm, equiangular_candidates(L)[perm]


# ---------------------------------------------------------------------------
# tables (transform.py:268-301, legendre.py:99-143)


@lru_cache(maxsize=8)
def packed_tables(L: int):
    """Packed recurrence factors (transform.py:268-291)."""
    size = L * (L + 1) // 2
    offsets = np.empty(L + 1, dtype=np.int64)
    a_curr = np.zeros(size)
    a_next = np.ones(size)
    pos = 0
    for m in range(L):
        offsets[m] = pos
        ells = np.arange(m, L, dtype=np.float64)
        a_curr[pos : pos + L - m] = np.sqrt((ells**2 - m * m) / ((2.0 * ells - 1.0) * (2.0 * ells + 1.0)))
        nxt = ells + 1.0
        a_next[pos : pos + L - m] = np.sqrt((nxt**2 - m * m) / ((2.0 * nxt - 1.0) * (2.0 * nxt + 1.0)))
        pos += L - m
    offsets[L] = pos
    q = np.arange(1, L + 1, dtype=np.float64)
    seed_fac = np.sqrt((2.0 * q - 1.0) / (2.0 * q))
    return offsets, a_curr, a_next, seed_fac


@lru_cache(maxsize=8)
def ring_roots_flat(L: int) -> np.ndarray:
    """exp(2 pi i r/(2k+1)) concatenated over rings (transform.py:294-301)."""
    return np.concatenate(
        [np.exp(2j * np.pi * np.arange(2 * k + 1) / (2 * k + 1)) for k in range(L)]
    )


def legendre_table(m: int, thetas, L: int) -> np.ndarray:
    """Y_lm(theta, 0) for l = |m|..L-1 (legendre.py:110-143)."""
    am = abs(m)
    if L < 1 or am >= L:
        raise ValueError(f"order {m} invalid for band limit {L}")
    thetas = np.ascontiguousarray(np.atleast_1d(np.asarray(thetas, dtype=np.float64)))
    ncols = L - am
    out = np.empty((thetas.size, ncols))
    seed0 = (-1.0) ** (am % 2) * math.sqrt((2 * am + 1) / FOUR_PI)
    q = np.arange(1, am + 1, dtype=np.float64)
    seed_fac = np.ascontiguousarray(np.sqrt((2.0 * q - 1.0) / (2.0 * q)))
    ells = np.arange(am, L, dtype=np.float64)
    a_curr = np.sqrt((ells**2 - am**2) / ((2.0 * ells - 1.0) * (2.0 * ells + 1.0)))
    en = ells + 1.0
    a_next = np.sqrt((en**2 - am**2) / ((2.0 * en - 1.0) * (2.0 * en + 1.0)))
    a_curr = np.ascontiguousarray(a_curr[: L - am - 1])
    a_next = np.ascontiguousarray(a_next[: L - am - 1])
    if a_curr.size == 0:  # keep valid pointers for the C call
        a_curr = np.zeros(1)
        a_next = np.ones(1)
    if seed_fac.size == 0:
        seed_fac = np.zeros(1)
    costh = np.ascontiguousarray(np.cos(thetas))
    sinth = np.ascontiguousarray(np.sin(thetas))
    _clib().oracle_legendre_kernel(
        _p(costh), _p(sinth), thetas.size, am, ncols, seed0, _p(seed_fac), _p(a_curr),
        _p(a_next), _p(out),
    )
    if m < 0 and am % 2:
        out = -out
    return out


# ---------------------------------------------------------------------------
# inverse (transform.py:304-357)


def synthesis_g(flm: np.ndarray, thetas: np.ndarray):
    """G_(+-m)(theta_k) as (L, L) complex matrices (transform.py:310-331)."""
    L = thetas.size
    offsets, a_curr, a_next, seed_fac = packed_tables(L)
    fcols = np.empty((L * (L + 1) // 2, 4))
    for m in range(L):
        ells = np.arange(m, L)
        fp = flm[ells * ells + ells + m]
        fn = flm[ells * ells + ells - m]
        sl = slice(offsets[m], offsets[m + 1])
        fcols[sl, 0] = fp.real
        fcols[sl, 1] = fp.imag
        fcols[sl, 2] = fn.real
        fcols[sl, 3] = fn.imag
    out = np.empty((L, L, 4))
    costh = np.ascontiguousarray(np.cos(thetas))
    sinth = np.ascontiguousarray(np.sin(thetas))
    _clib().oracle_g_accumulate(
        _p(costh), _p(sinth), L, _p(fcols), _p(seed_fac), _p(a_curr), _p(a_next),
        _p(offsets), L, _p(out),
    )
    out *= TWO_PI
    signs = np.ones(L)
    signs[1::2] = -1.0  # _order_signs, transform.py:304-307
    g_plus = out[:, :, 0] + 1j * out[:, :, 1]
    g_minus = (out[:, :, 2] + 1j * out[:, :, 3]) * signs[None, :]
    return g_plus, g_minus


def rings_from_tones(g_plus, g_minus, L: int) -> np.ndarray:
    """Fold tones into bins and inverse-FFT every ring (transform.py:334-344)."""
    bins = np.zeros(L * L, dtype=np.complex128)
    _clib().oracle_fold_bins(
        _p(np.ascontiguousarray(g_plus)), _p(np.ascontiguousarray(g_minus)), L, _p(bins)
    )
    out = np.empty(L * L, dtype=np.complex128)
    for k in range(L):
        n = 2 * k + 1
        s = k * k
        out[s : s + n] = (n / TWO_PI) * np.fft.ifft(bins[s : s + n])
    return out


def inverse_rings(flm: np.ndarray, thetas: np.ndarray, rings) -> dict:
    """inverse_sht restricted to the listed rings: {k: samples of ring k}.

    The same steps as inverse_sht (transform.py:347-357): _g_accumulate on the
    rings' co-latitudes only, then _fold_bins and the per-ring ifft for those
    rings -- O(L^2) per ring, so large-L rings can be checked one by one.
    """
    thetas = np.asarray(thetas, dtype=np.float64)
    L = thetas.size
    flm = np.asarray(flm, dtype=np.complex128)
    offsets, a_curr, a_next, seed_fac = packed_tables(L)
    fcols = np.empty((L * (L + 1) // 2, 4))
    for m in range(L):
        ells = np.arange(m, L)
        fp = flm[ells * ells + ells + m]
        fn = flm[ells * ells + ells - m]
        sl = slice(offsets[m], offsets[m + 1])
        fcols[sl, 0], fcols[sl, 1], fcols[sl, 2], fcols[sl, 3] = fp.real, fp.imag, fn.real, fn.imag
    rings = [int(k) for k in rings]
    th = thetas[rings]
    out = np.empty((len(rings), L, 4))
    _clib().oracle_g_accumulate(
        _p(np.ascontiguousarray(np.cos(th))), _p(np.ascontiguousarray(np.sin(th))), len(rings), _p(fcols),
        _p(seed_fac), _p(a_curr), _p(a_next), _p(offsets), L, _p(out),
    )
    out *= TWO_PI
    signs = np.ones(L)
    signs[1::2] = -1.0
    res = {}
    for i, k in enumerate(rings):
        n = 2 * k + 1
        gp = out[i, :, 0] + 1j * out[i, :, 1]
        gn = (out[i, :, 2] + 1j * out[i, :, 3]) * signs
        bins = np.zeros(n, dtype=np.complex128)
        for m in range(L):  # _fold_bins order (transform.py:204-218)
            bins[m % n] += gp[m]
            if m > 0:
                bins[(-m) % n] += gn[m]
        res[k] = (n / TWO_PI) * np.fft.ifft(bins)
    return res


def inverse_sht(flm: np.ndarray, thetas: np.ndarray) -> np.ndarray:
    """Flat complex128[L^2] coefficients -> flat ring-major samples (transform.py:347-357)."""
    thetas = np.asarray(thetas, dtype=np.float64)
    L = thetas.size
    flm = np.asarray(flm, dtype=np.complex128)
    if flm.size != L * L:
        raise ValueError("band limits disagree")
    g_plus, g_minus = synthesis_g(flm, thetas)
    return rings_from_tones(g_plus, g_minus, L)


# ---------------------------------------------------------------------------
# forward (transform.py:360-467, blocks.py:75-116)


def condition_number(entries: np.ndarray) -> float:
    """sigma_max/sigma_min (blocks.py:75-85)."""
    sv = np.linalg.svd(entries, compute_uv=False)
    if sv[-1] == 0.0 or not np.isfinite(sv[0]):
        return np.inf
    return float(sv[0] / sv[-1])


def solve_columns(entries, rhs, order, *, rcond=SOLVE_RCOND, check=True, driver="gelsy"):
    """Real-split gelsy solve with rank check (blocks.py:88-116).  ``driver`` other
    than gelsy is for tests only (the spread between two least-squares solvers)."""
    rhs = np.atleast_2d(rhs.T).T
    stacked = np.empty((entries.shape[0], 2 * rhs.shape[1]))
    stacked[:, 0::2] = rhs.real
    stacked[:, 1::2] = rhs.imag
    x, _, rank, _ = linalg.lstsq(entries, stacked, cond=rcond if check else None, lapack_driver=driver)
    if check and rank < entries.shape[1]:
        raise OracleIllConditioned(order, condition_number(entries))
    return x[:, 0::2] + 1j * x[:, 1::2]


def _solve_pair(block, g_p, g_n, m, sign, check):
    """transform.py:396-406 (timing bookkeeping omitted)."""
    if m == 0:
        f_p = solve_columns(block, g_p[:, None], 0, check=check)[:, 0]
        return f_p, f_p
    sol = solve_columns(block, np.column_stack([g_p, sign * g_n]), m, check=check)
    return sol[:, 0], sol[:, 1]


def forward_sht(samples: np.ndarray, thetas: np.ndarray, method: str = "direct",
                check: bool = True, stop_order: int = 0) -> np.ndarray:
    """Flat samples -> flat coefficients by top-down order peeling.

    ``method`` "direct" follows transform.py:409-433, "spectral" follows
    transform.py:436-467.  ``stop_order`` > 0 truncates the sweep after order
    ``stop_order`` (orders >= stop_order are exact);
    coefficients of lower orders are left zero.
    """
    thetas = np.asarray(thetas, dtype=np.float64)
    L = thetas.size
    samples = np.asarray(samples, dtype=np.complex128)
    if samples.size != L * L:
        raise ValueError("band limits disagree")
    if method not in ("direct", "spectral"):
        raise ValueError(f"unknown method {method!r}")
    coeffs = np.zeros(L * L, dtype=np.complex128)
    if method == "direct":
        buf = samples.copy()
        roots = ring_roots_flat(L)
    else:
        spectra = [np.fft.fft(samples[k * k : (k + 1) * (k + 1)]) for k in range(L)]
    lib = _clib()
    for m in range(L - 1, stop_order - 1, -1):
        table = legendre_table(m, thetas, L)
        g_p = np.empty(L - m, dtype=np.complex128)
        g_n = np.empty(L - m, dtype=np.complex128)
        if method == "direct":
            lib.oracle_peel_analyze(_p(buf), _p(roots), m, L, _p(g_p), _p(g_n))
        else:
            for k in range(m, L):
                n = 2 * k + 1
                delta = TWO_PI / n
                g_p[k - m] = delta * spectra[k][m % n]
                g_n[k - m] = delta * spectra[k][(-m) % n]
        sign = -1.0 if m % 2 else 1.0
        f_p, f_n = _solve_pair(TWO_PI * table[m:], g_p, g_n, m, sign, check)
        ells = np.arange(m, L)
        coeffs[ells * ells + ells + m] = f_p
        if m:
            coeffs[ells * ells + ells - m] = f_n
            cols = np.column_stack([f_p.real, f_p.imag, f_n.real, f_n.imag])
            gg = TWO_PI * (table[:m] @ cols)
            big_gp = np.ascontiguousarray(gg[:, 0] + 1j * gg[:, 1])
            big_gn = np.ascontiguousarray(sign * (gg[:, 2] + 1j * gg[:, 3]))
            if method == "direct":
                lib.oracle_peel_update(_p(buf), _p(roots), m, m, _p(big_gp), _p(big_gn))
            else:
                for k in range(m):
                    n = 2 * k + 1
                    spectra[k][m % n] -= n * big_gp[k] / TWO_PI
                    spectra[k][(-m) % n] -= n * big_gn[k] / TWO_PI
    return coeffs


def ring_analysis(ring_values, m: int):
    """Quadrature-exact (+m, -m) pair of one ring (transform.py:115-131)."""
    values = np.asarray(ring_values)
    n = values.shape[0]
    if n % 2 == 0:
        raise ValueError(f"ring length must be odd, got {n}")
    k = (n - 1) // 2
    if abs(m) > k:
        raise ValueError(f"frequency {m} is not resolvable on a ring of index {k}")
    spec = np.fft.fft(values)
    delta = TWO_PI / n
    return delta * spec[m % n], delta * spec[(-m) % n]


def block(m: int, thetas: np.ndarray) -> np.ndarray:
    """Order-m system 2*pi*Y_lm(theta_k, 0), k >= m (blocks.py:59-72)."""
    L = thetas.size
    return TWO_PI * legendre_table(m, thetas[m:], L)


def direct_synthesis(flm: np.ndarray, thetas: np.ndarray) -> np.ndarray:
    """Brute-force double sum at every sample (reference.py:26-65); small L only."""
    L = thetas.size
    tables = [legendre_table(m, thetas, L) for m in range(L)]
    out = np.empty(L * L, dtype=np.complex128)
    for k in range(L):
        n = 2 * k + 1
        phis = 2.0 * np.pi * np.arange(n) / n
        acc = np.zeros(n, dtype=np.complex128)
        for m in range(-(L - 1), L):
            am = abs(m)
            vals = tables[am][k]
            if m < 0 and am % 2:
                vals = -vals
            ells = np.arange(am, L)
            acc += np.exp(1j * m * phis) * (vals @ flm[ells * ells + ells + m])
        out[k * k : k * k + n] = acc
    return out


# ---------------------------------------------------------------------------
# BASELINE.json input recipes (SURVEY 8(d) "Generator convention")


def config_coefficients(L: int, rng, spectrum: str = "white", real: bool = False) -> np.ndarray:
    """One map: Re[L^2] then Im[L^2] N(0,1) in l^2+l+m order, then symmetry/scaling."""
    n = L * L
    f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    ells = np.floor(np.sqrt(np.arange(n))).astype(np.int64)
    ms = np.arange(n) - ells * ells - ells
    if real:
        f[ms == 0] = f[ms == 0].real
        neg = np.nonzero(ms < 0)[0]
        pos = ells[neg] ** 2 + ells[neg] - ms[neg]
        sgn = np.where((-ms[neg]) % 2 == 1, -1.0, 1.0)
        f[neg] = sgn * np.conj(f[pos])
    if spectrum == "cmb":
        cl = np.ones(n)
        nz = ells >= 1
        cl[nz] = 1.0 / (ells[nz] * (ells[nz] + 1.0))
        f = f * np.sqrt(cl)
    return f


# ---------------------------------------------------------------------------
# spin-weighted transforms (legendre.py:212-314, transform.py:474-533)

_BIG = 2.0**500  # legendre.py:31-36
_TINY = 2.0**-500
_UP = 2.0**1000
_DOWN = 2.0**-1000
_SHIFT = 1000


def spin_direct(spin: int, ell: int, m: int, theta: float) -> float:
    """sY_lm(theta, 0) from the explicit Wigner-d sum (legendre.py:175-218); small l only."""
    f = math.factorial
    m_row, m_col = -m, -spin  # spin_direct evaluates d^l_{-m,-s}
    if abs(m_row) > ell or abs(m_col) > ell:
        return 0.0
    ch, sh = math.cos(theta / 2.0), math.sin(theta / 2.0)
    pref = math.sqrt(f(ell + m_row) * f(ell - m_row) * f(ell + m_col) * f(ell - m_col))
    total = 0.0
    for k in range(max(0, m_col - m_row), min(ell + m_col, ell - m_row) + 1):
        num = ((-1.0) ** ((m_row - m_col + k) % 2) * ch ** (2 * ell + m_col - m_row - 2 * k)
               * sh ** (m_row - m_col + 2 * k))
        total += num / (f(ell + m_col - k) * f(k) * f(m_row - m_col + k) * f(ell - m_row - k))
    return (-1.0) ** (m % 2) * math.sqrt((2 * ell + 1) / FOUR_PI) * pref * total


def spin_seed_constants(spin: int, m: int):
    """(j, scale, offset, exp_sin, exp_cos) of the spin seed at l = j = max(|m|, |spin|)
    (legendre.py:233-262): scale = sign * sqrt(ratio2 / 2^shift2) * sqrt((2j+1)/4pi)
    from the exact rational ratio2, offset = shift2 / 2."""
    from fractions import Fraction

    j = max(abs(m), abs(spin))
    if j == 0:
        return 0, 1.0 / math.sqrt(FOUR_PI), 0, 0, 0
    k_lo = max(0, m - spin)
    k_hi = min(j - spin, j + m)
    assert k_lo == k_hi, "seed degree must sit at a corner of the d-matrix"
    k = k_lo
    exp_sin = spin - m + 2 * k
    exp_cos = 2 * j - exp_sin
    sign = -1.0 if (k + spin) % 2 else 1.0
    f = math.factorial
    numer = f(j - m) * f(j + m) * f(j - spin) * f(j + spin)
    denom = f(j - spin - k) * f(k) * f(spin - m + k) * f(j + m - k)
    ratio2 = Fraction(numer, denom * denom)
    shift2 = ratio2.numerator.bit_length() - ratio2.denominator.bit_length()
    if shift2 % 2:
        shift2 -= 1
    base = math.sqrt(float(ratio2 / Fraction(2) ** shift2))
    scale = sign * base * math.sqrt((2 * j + 1) / FOUR_PI)
    return j, scale, shift2 // 2, exp_sin, exp_cos


def _rescale_small(mant, off):
    lo = (np.abs(mant) < _TINY) & (mant != 0.0)
    mant[lo] *= _UP
    off[lo] -= _SHIFT


def _rescale_pair(curr, prev, off):
    hi = np.abs(curr) > _BIG
    curr[hi] *= _DOWN
    prev[hi] *= _DOWN
    off[hi] += _SHIFT
    lo = (np.abs(curr) < _TINY) & (np.abs(prev) < _TINY) & ((curr != 0.0) | (prev != 0.0))
    curr[lo] *= _UP
    prev[lo] *= _UP
    off[lo] -= _SHIFT


def spin_table(spin: int, m: int, thetas, L: int) -> np.ndarray:
    """sY_lm(theta, 0) for l = max(|m|, |spin|)..L-1, shape (len(thetas), L - lo)
    (legendre.py:276-314: exact-rational seed, rescaled three-term recurrence)."""
    lo = max(abs(m), abs(spin))
    if L < 1 or lo >= L:
        raise ValueError(f"order {m}, spin {spin} invalid for band limit {L}")
    thetas = np.atleast_1d(np.asarray(thetas, dtype=np.float64))
    costh = np.cos(thetas)
    out = np.empty((thetas.size, L - lo))
    j, scale, off0, exp_sin, exp_cos = spin_seed_constants(spin, m)
    mant = np.full(thetas.size, scale)
    off = np.full(thetas.size, off0, dtype=np.int64)
    ch, sh = np.cos(thetas / 2.0), np.sin(thetas / 2.0)
    for _ in range(exp_sin):
        mant *= sh
        _rescale_small(mant, off)
    for _ in range(exp_cos):
        mant *= ch
        _rescale_small(mant, off)
    out[:, 0] = np.ldexp(mant, off)
    prev = np.zeros_like(mant)
    curr = mant
    ms = float(m * spin)
    for idx, ell in enumerate(range(lo, L - 1)):
        if ell == 0:
            nxt = math.sqrt(3.0) * costh * curr
        else:
            d = ell * math.sqrt(((ell + 1.0) ** 2 - m * m) * ((ell + 1.0) ** 2 - spin * spin) / (2 * ell + 3))
            a = math.sqrt(2 * ell + 1.0) * ell * (ell + 1.0)
            b = math.sqrt(2 * ell + 1.0) * ms
            c = (ell + 1.0) * math.sqrt((ell * ell - m * m) * (ell * ell - spin * spin) / (2 * ell - 1.0))
            nxt = ((a * costh - b) * curr - c * prev) / d
        prev = curr
        curr = nxt
        _rescale_pair(curr, prev, off)
        out[:, idx + 1] = np.ldexp(curr, off)
    return out


def spin_inverse_sht(flm: np.ndarray, thetas: np.ndarray, spin: int) -> np.ndarray:
    """Spin-weighted synthesis (transform.py:474-496); degrees below |spin| ignored."""
    thetas = np.asarray(thetas, dtype=np.float64)
    L = thetas.size
    flm = np.asarray(flm, dtype=np.complex128)
    if abs(spin) >= L:
        raise ValueError(f"spin {spin} invalid for band limit {L}")
    if spin == 0:
        return inverse_sht(flm, thetas)
    g_plus = np.empty((L, L), dtype=np.complex128)
    g_minus = np.empty((L, L), dtype=np.complex128)
    for m in range(L):
        lo = max(m, abs(spin))
        ells = np.arange(lo, L)
        g_plus[:, m] = TWO_PI * (spin_table(spin, m, thetas, L) @ flm[ells * ells + ells + m])
        g_minus[:, m] = TWO_PI * (spin_table(spin, -m, thetas, L) @ flm[ells * ells + ells - m])
    return rings_from_tones(g_plus, g_minus, L)


def spin_forward_sht(samples: np.ndarray, thetas: np.ndarray, spin: int, check: bool = True,
                     driver: str = "gelsy") -> np.ndarray:
    """Spin-weighted analysis by top-down peeling (transform.py:499-533): per order the
    +m and -m blocks 2pi sY_l(+-m)(theta_k), k >= |m|, are solved separately (tall for
    |m| < |spin|, least squares); degrees below |spin| come back zero."""
    thetas = np.asarray(thetas, dtype=np.float64)
    L = thetas.size
    samples = np.asarray(samples, dtype=np.complex128)
    if abs(spin) >= L:
        raise ValueError(f"spin {spin} invalid for band limit {L}")
    if spin == 0:
        return forward_sht(samples, thetas, check=check)
    coeffs = np.zeros(L * L, dtype=np.complex128)
    buf = samples.copy()
    roots = ring_roots_flat(L)
    lib = _clib()
    for m in range(L - 1, -1, -1):
        lo = max(m, abs(spin))
        tab_p = spin_table(spin, m, thetas, L)
        tab_n = spin_table(spin, -m, thetas, L)
        g_p = np.empty(L - m, dtype=np.complex128)
        g_n = np.empty(L - m, dtype=np.complex128)
        lib.oracle_peel_analyze(_p(buf), _p(roots), m, L, _p(g_p), _p(g_n))
        f_p = solve_columns(TWO_PI * tab_p[m:], g_p[:, None], m, check=check, driver=driver)[:, 0]
        f_n = f_p if m == 0 else solve_columns(TWO_PI * tab_n[m:], g_n[:, None], -m, check=check,
                                               driver=driver)[:, 0]
        ells = np.arange(lo, L)
        coeffs[ells * ells + ells + m] = f_p
        if m:
            coeffs[ells * ells + ells - m] = f_n
            big_gp = np.ascontiguousarray(TWO_PI * (tab_p[:m] @ f_p))
            big_gn = np.ascontiguousarray(TWO_PI * (tab_n[:m] @ f_n))
            lib.oracle_peel_update(_p(buf), _p(roots), m, m, _p(big_gp), _p(big_gn))
    return coeffs
