"""Per-order blocks and their solves: the public API of the reference's
blocks.py (LegendreBlock / GVector / CoefficientSlice, block_for_thetas,
build_block, condition_number, solve; blocks.py:30-140).

The transforms never call this module -- libosph factors every block itself
(pivots.cu, factor_bf.cu).  It serves callers that inspect single blocks:
entries are generated on the device (legendre.legendre_table), the
condition number and the solve use torch.linalg on the GPU (singular values;
QR least squares with a singular-value rank test at rcond, standing in for
gelsy's rank-revealing QR).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import IllConditionedSolveError, OrderRangeError
from .legendre import legendre_table

TWO_PI = 2.0 * np.pi
SOLVE_RCOND = 1e-14  # blocks.py:27


@dataclass(frozen=True)
class LegendreBlock:
    """Square synthesis block for one order, rows following the grid suffix (blocks.py:30-40)."""

    order: int
    sign: int
    entries: np.ndarray

    @property
    def size(self) -> int:
        return self.entries.shape[0]


@dataclass(frozen=True)
class GVector:
    """Ring-integrated Fourier content G_m(theta_k) over a grid suffix (blocks.py:43-48)."""

    order: int
    values: np.ndarray


@dataclass(frozen=True)
class CoefficientSlice:
    """Harmonic coefficients of one order, degrees |m| .. L-1 (blocks.py:51-56)."""

    order: int
    values: np.ndarray


def block_for_thetas(m: int, thetas, band_limit: int, device: int = 0) -> LegendreBlock:
    """The order-m block on explicit ring co-latitudes (blocks.py:59-64)."""
    am = abs(int(m))
    entries = TWO_PI * legendre_table(am, thetas, band_limit, device)
    return LegendreBlock(order=am, sign=-1 if (m < 0 and am % 2) else 1, entries=entries)


def build_block(grid, m: int, device: int = 0) -> LegendreBlock:
    """The order-m block on the suffix rings |m| .. L-1 of a grid (blocks.py:67-72)."""
    am = abs(int(m))
    if am >= grid.band_limit:
        raise OrderRangeError(f"order {m} invalid for band limit {grid.band_limit}")
    return block_for_thetas(m, grid.thetas[am:], grid.band_limit, device)


def _singular_values(a: np.ndarray, device: int):
    import torch

    return torch.linalg.svdvals(torch.as_tensor(np.asarray(a, dtype=np.float64), device=f"cuda:{device}")).cpu().numpy()


def condition_number(block, device: int = 0) -> float:
    """sigma_max / sigma_min; infinity when singular (blocks.py:75-85)."""
    entries = block.entries if isinstance(block, LegendreBlock) else np.asarray(block)
    sv = _singular_values(entries, device)
    if sv[-1] == 0.0 or not np.isfinite(sv[0]):
        return np.inf
    return float(sv[0] / sv[-1])


def solve(block: LegendreBlock, g, *, rcond: float = SOLVE_RCOND, check: bool = True,
          device: int = 0) -> CoefficientSlice:
    """f with block * f = g (blocks.py:119-140): GVector or plain array; the
    stored sign of a negative order is folded into the right-hand side.
    check: rank < n at rcond (singular values) -> IllConditionedSolveError."""
    import torch

    if isinstance(g, GVector):
        order = g.order
        values = np.asarray(g.values, dtype=np.complex128)
    else:
        order = block.order if block.sign == 1 else -block.order
        values = np.asarray(g, dtype=np.complex128)
    if values.shape[0] != block.size:
        raise ValueError(f"right-hand side length {values.shape[0]} does not match block size {block.size}")
    a = np.asarray(block.entries, dtype=np.float64)
    if check:
        sv = _singular_values(a, device)
        if not (sv[-1] > rcond * sv[0]) or a.shape[0] < a.shape[1]:
            raise IllConditionedSolveError(order, np.inf if sv[-1] == 0.0 else float(sv[0] / sv[-1]))
    rhs = block.sign * values
    dev = f"cuda:{device}"
    stacked = np.stack([rhs.real, rhs.imag], axis=1)  # real-split columns (blocks.py:110-116)
    x = torch.linalg.lstsq(torch.as_tensor(a, device=dev), torch.as_tensor(stacked, device=dev)).solution
    x = x.cpu().numpy()
    return CoefficientSlice(order=order, values=x[:, 0] + 1j * x[:, 1])
