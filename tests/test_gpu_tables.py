"""GPU: the reference's public table and block API (legendre.py:39-150,
276-314; blocks.py:30-140) served by the device kernels -- against the
reference's own tables (tests/golden/ref_L*.npz) and the oracle."""

import numpy as np
import pytest

from conftest import GOLDEN, GRIDS, has_gpu
from oracle import optisph_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.mark.parametrize("L,ms", [(16, (0, 1, 8, 15)), (64, (0, 1, 32, 63))])
def test_legendre_table_matches_reference(L, ms):
    import paper_1403_4661_b200 as osp

    ref = np.load(GOLDEN / f"ref_L{L}.npz")
    for m in ms:
        got = osp.legendre_table(m, ref["thetas"], L)
        want = ref[f"table_m{m}"]
        assert got.shape == want.shape
        assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def test_legendre_table_signs_columns_and_range():
    import paper_1403_4661_b200 as osp

    th = np.linspace(0.05, np.pi, 50)  # more co-latitudes than L: several plans
    for m in (-5, -4, 3):
        assert np.abs(osp.legendre_table(m, th, 20) - O.legendre_table(m, th, 20)).max() <= 1e-12
    col = osp.legendre_column(-3, 0.7, 12)
    assert col.order == -3 and col.value(5) == pytest.approx(O.legendre_table(-3, [0.7], 12)[0][2], abs=1e-13)
    sc = osp.spin_column(2, -1, 1.3, 10)
    assert sc.value(4) == pytest.approx(O.spin_table(2, -1, [1.3], 10)[0][2], abs=1e-13)
    with pytest.raises(osp.OrderRangeError):
        osp.legendre_table(12, th, 12)


@pytest.mark.parametrize("m", [0, 5, -7, 40])
def test_blocks_and_solve_match_oracle(grid_of, m):
    import paper_1403_4661_b200 as osp

    grid = grid_of(64)
    blk = osp.build_block(grid, m)
    want = O.block(abs(m), grid.thetas)
    assert blk.order == abs(m) and blk.sign == (-1 if (m < 0 and abs(m) % 2) else 1)
    assert np.abs(blk.entries - want).max() <= 1e-12 * np.abs(want).max()
    assert osp.condition_number(blk) == pytest.approx(O.condition_number(want), rel=1e-9)
    rng = np.random.default_rng(7)
    g = rng.standard_normal(blk.size) + 1j * rng.standard_normal(blk.size)
    x = osp.solve(blk, g)
    ref = O.solve_columns(want, (blk.sign * g)[:, None], m)[:, 0]
    assert x.order == m
    assert np.abs(x.values - ref).max() <= 1e-11 * max(1.0, np.abs(ref).max())
    gv = osp.solve(blk, osp.GVector(order=m, values=g))
    assert np.array_equal(gv.values, x.values)


def test_solve_refuses_the_singular_block_like_the_reference():
    import paper_1403_4661_b200 as osp

    misc = np.load(GOLDEN / "ref_misc.npz")
    order = int(misc["illcond_order"])
    grid = osp.load_grid(GRIDS / "grid-L256-uniform-interleaved.txt")
    blk = osp.build_block(grid, order)
    with pytest.raises(osp.IllConditionedSolveError) as ei:
        osp.solve(blk, np.ones(blk.size))
    assert ei.value.order == order
    osp.solve(blk, np.ones(blk.size), check=False)  # least squares without the rank test
