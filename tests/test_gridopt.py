"""Grid optimiser (gridopt.py): rank-one secular kappa and the greedy, checked on CPU.

The greedy's Legendre rows come from the oracle here (the GPU run uses
osph_legendre_block); the permutations must equal the reference's own
condition-minimised grids (tests/golden/grids, written by the reference's
optimize_order, sampling.py:217-278).
"""

import numpy as np
import pytest
import torch

from oracle import optisph_oracle as O
from paper_1403_4661_b200 import gridopt, sampling


def test_rank_one_kappas_match_svd():
    rng = np.random.default_rng(3)
    for n in (2, 3, 7, 40):
        A0 = rng.standard_normal((n - 1, n))
        R = rng.standard_normal((9, n))
        d, V = np.linalg.eigh(A0.T @ A0)
        k = gridopt.rank_one_kappas(torch.from_numpy(d), torch.from_numpy(R @ V)).numpy()
        ref = [np.linalg.cond(np.vstack([r[None, :], A0])) for r in R]
        np.testing.assert_allclose(k, ref, rtol=1e-10)


def test_rank_one_kappas_singular_is_inf():
    rng = np.random.default_rng(4)
    A0 = rng.standard_normal((4, 5))
    r = A0[1] * 2.0 - A0[3]  # in the row space: the stacked block is singular
    d, V = np.linalg.eigh(A0.T @ A0)
    k = gridopt.rank_one_kappas(torch.from_numpy(d), torch.from_numpy((r @ V)[None, :])).numpy()
    assert k[0] > 1e12


@pytest.mark.parametrize("L", [8, 16, 32, 64])
def test_greedy_reproduces_reference_grids(L, grid_of):
    cands = sampling.equiangular_candidates(L)
    perm = gridopt.greedy_order(L, lambda m: torch.from_numpy(O.legendre_table(m, cands, L)))
    assert np.array_equal(perm, grid_of(L).permutation)
