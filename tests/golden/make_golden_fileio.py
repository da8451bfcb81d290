"""Coefficient/signal files written by the REFERENCE's fileio (fileio.py:28-47), for format parity.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_fileio.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import optisph as osp  # noqa: E402
from optisph import fileio  # noqa: E402

OUT = Path(__file__).resolve().parent / "fileio"
OUT.mkdir(exist_ok=True)
L = 4
rng = np.random.default_rng(4661)
f = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
f[0] = -0.0 + 1e-300j  # signed zero and a tiny value through the 17-digit format
fileio.write_coefficients(OUT / "coef_L4.txt", osp.HarmonicCoefficients(L, f))
s = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
fileio.write_signal(OUT / "sig_L4.txt", osp.SpatialSamples.from_flat(L, s))
np.savez(OUT / "values_L4.npz", flm=f, samples=s)
print("wrote", OUT)
