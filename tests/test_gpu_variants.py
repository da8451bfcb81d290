"""GPU: the factorisation's kernel variants give bit-identical coefficients.

The breadth-first update runs on 64 x 64 or 128 x 64 tiles (chosen by L,
forced by OSPH_BF_UPD_ROWS), and the next step's R panel is either handed
off by the panel and update kernels or copied by its own launch
(OSPH_BF_RFUSE=0); the orders are factored as one chain or as several
ranges on their own streams (OSPH_FACTOR_SPLIT).  Every variant performs the same DMMA chain per element,
so the forward output must not change by a single bit.  The switches are
read once per process, so each variant runs in a subprocess; the default
result is also checked against the round-trip bar of the other parity tests.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1403_4661_b200 as osp
L, B, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
grid = osp.load_grid(sys.argv[1] + f"/tests/golden/grids/grid-L{L}-uniform-condmin.txt")
rng = np.random.default_rng(L)
samples = rng.standard_normal((B, L * L)) + 1j * rng.standard_normal((B, L * L))
flm = osp.forward_sht_batch(samples, grid, check=False)
rt = osp.forward_sht_batch(osp.inverse_sht_batch(flm, grid), grid, check=False)
np.savez(out, flm=flm, rt_err=np.abs(rt - flm).max())
"""

VARIANTS = [{}, {"OSPH_BF_UPD_ROWS": "64"}, {"OSPH_BF_UPD_ROWS": "128"}, {"OSPH_BF_RFUSE": "0"},
            {"OSPH_BF_UPD_ROWS": "128", "OSPH_BF_RFUSE": "0"},
            # the factorisation as one chain / four order ranges on their own streams (default three)
            {"OSPH_FACTOR_SPLIT": "0"}, {"OSPH_FACTOR_SPLIT": "4"}]


def run_variant(tmp_path, L, B, env_extra, tag):
    out = tmp_path / f"v_{L}_{tag}.npz"
    env = dict(os.environ)
    env.update(env_extra)
    subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), str(L), str(B), str(out)], env=env, check=True,
                   timeout=600)
    return np.load(out)


@pytest.mark.parametrize("L,B", [(256, 2), (512, 1), (2048, 1)])
def test_factor_variants_bit_identical(tmp_path, L, B):
    base = run_variant(tmp_path, L, B, VARIANTS[0], 0)
    # round trip of a random (not band-limited) map's coefficients; L = 2048: DESIGN 6's chain amplification
    assert float(base["rt_err"]) <= (1e-9 if L <= 512 else 0.12)
    for i, v in enumerate(VARIANTS[1:], 1):
        got = run_variant(tmp_path, L, B, v, i)
        assert np.array_equal(got["flm"], base["flm"]), f"variant {v} differs: " \
            f"{np.abs(got['flm'] - base['flm']).max():.3e}"


@pytest.mark.parametrize("L,B", [(256, 2), (512, 1), (2048, 1)])
def test_paired_steps_match_single_steps(tmp_path, L, B):
    """Paired (rank-128) breadth-first steps against rank-64 steps: the same elimination
    in a different association order, so equal to rounding (L = 2048: on the orders the
    peeling chain has not yet amplified, m >= L/2; DESIGN 6)."""
    single = run_variant(tmp_path, L, B, {"OSPH_BF_PAIR": "0"}, "single")
    paired = run_variant(tmp_path, L, B, {"OSPH_BF_PAIR": "1"}, "paired")
    assert float(paired["rt_err"]) <= (1e-9 if L <= 512 else 0.12)
    a, b = paired["flm"], single["flm"]
    if L >= 2048:
        ell = np.floor(np.sqrt(np.arange(L * L))).astype(np.int64)
        m = np.abs(np.arange(L * L) - ell * ell - ell)
        keep = m >= L // 2
        a, b = a[:, keep], b[:, keep]
    scale = max(1.0, float(np.abs(b).max()))
    assert np.abs(a - b).max() <= 1e-11 * scale, f"{np.abs(a - b).max():.3e} vs scale {scale:.3e}"
