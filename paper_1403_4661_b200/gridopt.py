"""Condition-minimising ring order on the GPU: ``optimize_order`` for large L.

The reference's greedy (sampling.py:217-278) pins the largest ring to the
candidate nearest the equator (index (L-1)//2 for the uniform measure), then
walks m = L-2 .. 0 and gives ring m the unassigned candidate t that minimises
the 2-norm condition number of the order-m block on the suffix
{theta_t, theta_perm[m+1], ..., theta_perm[L-1]} (blocks.py:60-85); near ties
(relative 1e-9) go to the candidate nearest the equator, then the lower index.
Done literally that is one n x n SVD per candidate, O(L^5) in total (1,306 s at
L=512 on one core).

Here every step factors the block of the chosen rings once.  With
A0 ((n-1) x n, the chosen rings' rows of Y_lm, l = m..L-1) and
A0^T A0 = V diag(d) V^T, the block of candidate t is A = [r_t; A0] and

    A^T A = V (diag(d) + z z^T) V^T,   z = V^T r_t,

so its squared singular values are the roots of the secular equation
1 + sum_i z_i^2 / (d_i - lambda) = 0, whose smallest and largest roots lie in
[d_0, d_1] and [d_{n-1}, d_{n-1} + |z|^2] (interlacing) and are found by
bisection for all candidates at once.  Row order does not change singular
values, so kappa(t) = sqrt(lambda_max / lambda_min) is the reference's
kappa.  Cost per step: one Gram GEMM + one symmetric eigendecomposition
(O(n^3), cuBLAS/cuSOLVER through torch -- this is an offline setup tool, not
the transform path) + one candidates x n GEMM + O(c n) bisection sweeps.
The Legendre rows of all L candidates come from the library's on-device
recurrence (``osph_legendre_block``).

kappa agrees with the reference's SVD to about eps * kappa^2 relative (the
Gram squares the spread), far inside the 1e-9 tie tolerance for the
condition numbers of these grids (kappa <= a few hundred at L <= 512, SURVEY
A.5); the output is checked against the reference's own L <= 512 grids.
"""

from __future__ import annotations

import argparse
import ctypes
import time

import numpy as np

from . import _lib
from .errors import OptisphError
from .sampling import ColatitudeGrid, equiangular_candidates, grid_from_permutation, save_grid


class IllConditionedGridError(OptisphError, RuntimeError):
    """No candidate gives a finite condition number at this order (errors.py IllConditionedGridError)."""

    def __init__(self, order: int):
        super().__init__(f"no well-conditioned candidate for order {order}")
        self.order = order


def rank_one_kappas(d, Z, iters: int = 160):
    """kappa_2 of [r; A0] for every row r of ``R`` given A0^T A0 = V diag(d) V^T and Z = R V.

    ``d`` ascending (n,), ``Z`` (c, n); torch tensors on any device.  Returns a
    (c,) tensor, +inf where the block is singular.
    """
    import torch

    d = torch.clamp(d, min=0.0)
    z2 = Z * Z
    c, n = z2.shape
    if n == 1:
        lam = d[0] + z2[:, 0]
        return torch.where(lam > 0, torch.ones_like(lam), torch.full_like(lam, float("inf")))

    def root(lo, hi):
        # f(lambda) = 1 + sum z_i^2 / (d_i - lambda) is increasing between poles
        for _ in range(iters):
            mid = 0.5 * (lo + hi)
            f = 1.0 + (z2 / (d[None, :] - mid[:, None])).sum(dim=1)
            neg = f < 0
            lo = torch.where(neg, mid, lo)
            hi = torch.where(neg, hi, mid)
        return 0.5 * (lo + hi)

    lo = d[0].expand(c).clone()
    hi = d[1].expand(c).clone()
    lam_min = root(lo, hi)
    lo = d[-1].expand(c).clone()
    hi = d[-1] + z2.sum(dim=1)
    lam_max = root(lo, hi)
    kap = torch.sqrt(lam_max / lam_min)
    bad = ~(lam_min > 0) | ~torch.isfinite(kap)
    return torch.where(bad, torch.full_like(kap, float("inf")), kap)


def greedy_order(L: int, rows_of, *, tie_rtol: float = 1e-9, progress=None) -> np.ndarray:
    """The reference's greedy with the rank-one kappa evaluation.

    ``rows_of(m)`` returns a torch tensor (L, L-m): row j = Y_lm(cand_j), l = m..L-1,
    for the L equiangular candidates.  Returns perm (int64[L]).
    """
    import torch

    cands = equiangular_candidates(L)
    equator_dist = np.abs(cands - np.pi / 2.0)  # sampling.py:256
    perm = np.empty(L, dtype=np.int64)
    unassigned = list(range(L))
    first = (L - 1) // 2
    perm[L - 1] = first
    unassigned.remove(first)
    t0 = time.time()
    for m in range(L - 2, -1, -1):
        P = rows_of(m)
        dev = P.device
        chosen = torch.as_tensor(perm[m + 1:], device=dev)
        A0 = P.index_select(0, chosen)
        G = A0.T @ A0
        d, V = torch.linalg.eigh(G)
        R = P.index_select(0, torch.as_tensor(unassigned, device=dev))
        kappas = rank_one_kappas(d, R @ V).cpu().numpy()
        best = np.min(kappas)
        if not np.isfinite(best):
            raise IllConditionedGridError(m)
        near = kappas <= best * (1.0 + tie_rtol)
        ranked = sorted((equator_dist[t], t) for i, t in enumerate(unassigned) if near[i])
        pick = ranked[0][1]
        perm[m] = pick
        unassigned.remove(pick)
        if progress is not None and (m % progress == 0):
            print(f"[gridopt] L={L} m={m} kappa={best:.6g} ({time.time() - t0:.1f} s)", flush=True)
    return perm


def optimize_order(band_limit: int, device: int = 0, *, tie_rtol: float = 1e-9, progress=None) -> ColatitudeGrid:
    """Condition-minimised uniform grid for ``band_limit`` (sampling.py:217-278), on ``device``."""
    import torch

    L = int(band_limit)
    cands = equiangular_candidates(L)
    lib = _lib.load()
    handle = ctypes.c_void_p()
    th = np.ascontiguousarray(cands)
    devs = (ctypes.c_int * 1)(device)
    _lib.raise_for(lib.osph_plan_create(L, th.ctypes.data_as(ctypes.c_void_p), 1, 1, ctypes.cast(devs, ctypes.c_void_p),
                                        ctypes.byref(handle)))
    try:
        buf = torch.empty((L, L), dtype=torch.float64, device=f"cuda:{device}")

        def rows_of(m: int):
            _lib.raise_for(lib.osph_legendre_block(handle, m, ctypes.c_void_p(buf.data_ptr()), L,
                                                   _lib.OSPH_DEVICE))
            return buf[: L - m].T  # (candidates, degrees)

        perm = greedy_order(L, rows_of, tie_rtol=tie_rtol, progress=progress)
    finally:
        lib.osph_plan_destroy(handle)
    return grid_from_permutation(L, perm)


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description="condition-minimised uniform grid on the GPU")
    ap.add_argument("L", type=int)
    ap.add_argument("out")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--progress", type=int, default=256)
    args = ap.parse_args(argv)
    t0 = time.time()
    grid = optimize_order(args.L, args.device, progress=args.progress)
    save_grid(grid, args.out)
    print(f"[gridopt] L={args.L} written to {args.out} in {time.time() - t0:.1f} s", flush=True)


# ---------------------------------------------------------------------------
# reference-shaped entry points (sampling.py:217-313)


def optimize_order_like_reference(cands, band_limit: int, block_builder=None, measure=None,
                                  tie_rtol: float = 1e-9, device: int = 0) -> ColatitudeGrid:
    """``optimize_order(cands, band_limit, ...)`` with the reference's signature.

    Only the uniform measure's equiangular candidates are on this package's
    path; a custom ``block_builder`` is not supported (the blocks are built on
    the device).
    """
    from .sampling import Measure

    if measure not in (None, Measure.UNIFORM):
        raise NotImplementedError("only the uniform measure is supported")
    if block_builder is not None:
        raise NotImplementedError("custom block builders are not supported (blocks are built on the GPU)")
    if not np.array_equal(np.asarray(cands, dtype=np.float64), equiangular_candidates(band_limit)):
        raise ValueError("candidates must be the uniform measure's equiangular candidates")
    return optimize_order(band_limit, device, tie_rtol=tie_rtol)


def make_grid(band_limit: int, measure=None, ordering=None, cache_dir=None, device: int = 0) -> ColatitudeGrid:
    """``make_grid`` (sampling.py:281-313): interleaved, or condition-minimised with an on-disk cache."""
    from pathlib import Path

    from .sampling import Measure, Ordering, interleaved_grid, load_grid

    measure = Measure.UNIFORM if measure is None else measure
    ordering = Ordering.INTERLEAVED if ordering is None else ordering
    if measure is not Measure.UNIFORM:
        raise NotImplementedError("only the uniform measure is supported")
    if ordering is Ordering.INTERLEAVED:
        return interleaved_grid(band_limit)
    path = None
    if cache_dir is not None:
        path = Path(cache_dir) / f"grid-L{band_limit}-{measure.value}-{ordering.value}.txt"
        if path.exists():
            grid = load_grid(path)
            if grid.band_limit == band_limit and grid.ordering is ordering:
                return grid
    grid = optimize_order(band_limit, device)
    if path is not None:
        path.parent.mkdir(parents=True, exist_ok=True)
        save_grid(grid, path)
    return grid


if __name__ == "__main__":
    main()
