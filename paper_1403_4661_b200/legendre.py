"""Basis tables on the device: the public table API of the reference's
legendre.py (legendre_table / legendre_column / spin_table / spin_column and
their dataclasses, legendre.py:39-61, 110-150, 276-314).

Every value comes from libosph's recurrence kernels (osph_legendre_block,
osph_spin_block), evaluated on plans whose rings are the requested
co-latitudes, L at a time (a plan needs L co-latitudes in (0, pi]; a short
last chunk is padded with pi/2 and the padding rows dropped).  Values below
2^-500 come back as 0 (the reference returns the denormal-range value
itself, < 2^-500 in magnitude).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import OrderRangeError


@dataclass(frozen=True)
class LegendreColumn:
    """Values Y_lm(theta, 0) for ell = |order| .. L-1 at one co-latitude (legendre.py:39-48)."""

    order: int
    theta: float
    values: np.ndarray

    def value(self, ell: int) -> float:
        return self.values[ell - abs(self.order)]


@dataclass(frozen=True)
class SpinColumn:
    """Spin-weighted values at longitude zero, ell = max(|order|, |spin|) .. L-1 (legendre.py:51-61)."""

    spin: int
    order: int
    theta: float
    values: np.ndarray

    def value(self, ell: int) -> float:
        return self.values[ell - max(abs(self.order), abs(self.spin))]


def _device_table(fill, thetas, L: int, rows: int, device: int) -> np.ndarray:
    """(len(thetas), rows) table; fill(plan, out_ptr, ld) writes [degree][ring] on the device."""
    import torch

    from .transform import get_plan

    th = np.atleast_1d(np.asarray(thetas, dtype=np.float64))
    if th.size and not (np.all(th > 0.0) and np.all(th <= np.pi)):
        raise ValueError("co-latitudes must lie in (0, pi]")
    out = np.empty((th.size, rows))
    buf = torch.empty((max(rows, 1), L), dtype=torch.float64, device=f"cuda:{device}")
    for c0 in range(0, th.size, L):
        chunk = th[c0:c0 + L]
        padded = np.concatenate([chunk, np.full(L - chunk.size, np.pi / 2)])
        plan = get_plan(padded, 1, device)
        with plan.lock:
            plan.set_stream(None)
            fill(plan, buf.data_ptr(), L)  # synchronous on the plan stream
        out[c0:c0 + chunk.size] = buf[:rows].cpu().numpy().T[: chunk.size]
    return out


def legendre_table(m: int, thetas, band_limit: int, device: int = 0) -> np.ndarray:
    """Y_lm(theta, 0), shape (len(thetas), L - |m|); column j is degree |m| + j.
    Negative orders apply Y_l(-m) = (-1)^m Y_lm (legendre.py:110-143)."""
    L = int(band_limit)
    am = abs(int(m))
    if L < 1 or am >= L:
        raise OrderRangeError(f"order {m} invalid for band limit {L}")

    def fill(plan, ptr, ld):
        _lib.raise_for(plan._lib.osph_legendre_block(plan.handle, am, ctypes.c_void_p(ptr), ld, _lib.OSPH_DEVICE))

    out = _device_table(fill, thetas, L, L - am, device)
    if m < 0 and am % 2:
        out = -out
    return out


def legendre_column(m: int, theta: float, band_limit: int, device: int = 0) -> LegendreColumn:
    """Single-point legendre_table (legendre.py:146-150)."""
    return LegendreColumn(order=m, theta=float(theta), values=legendre_table(m, [theta], band_limit, device)[0])


def spin_table(spin: int, m: int, thetas, band_limit: int, device: int = 0) -> np.ndarray:
    """sY_lm(theta, 0) for l = max(|m|, |spin|)..L-1, shape (len(thetas), L - lo)
    (legendre.py:276-306: exact-rational seed, rescaled recurrence; osph_spin_block)."""
    L = int(band_limit)
    lo = max(abs(int(m)), abs(int(spin)))
    if L < 1 or lo >= L:
        raise OrderRangeError(f"order {m}, spin {spin} invalid for band limit {L}")

    def fill(plan, ptr, ld):
        plan.spin_block(spin, m, ptr, ld)

    return _device_table(fill, thetas, L, L - lo, device)


def spin_column(spin: int, m: int, theta: float, band_limit: int, device: int = 0) -> SpinColumn:
    """Single-point spin_table (legendre.py:309-314)."""
    return SpinColumn(spin=spin, order=m, theta=float(theta),
                      values=spin_table(spin, m, [theta], band_limit, device)[0])
