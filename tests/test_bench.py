"""bench.py helpers on CPU: input recipes, work counts, the CPU-baseline estimator."""

import numpy as np

import bench
from oracle import optisph_oracle as O


def test_recipes_match_oracle_generator():
    # BASELINE recipes: the bench and the oracle/fixtures draw identical maps
    for spectrum, real in [("white", False), ("cmb", False), ("cmb", True)]:
        got = bench.make_coefficients(16, 3, 42, spectrum, real)
        rng = np.random.default_rng(42)
        want = np.stack([O.config_coefficients(16, rng, spectrum=spectrum, real=real) for _ in range(3)])
        assert np.array_equal(got, want)


def test_real_recipe_is_conjugate_symmetric():
    L = 12
    f = bench.make_coefficients(L, 1, 3, "cmb", True)[0]
    for l in range(L):
        for m in range(1, l + 1):
            assert f[l * l + l - m] == (-1) ** m * np.conj(f[l * l + l + m])
        assert f[l * l + l].imag == 0.0


def test_flop_counts():
    fl = bench.flops(256, 64)
    assert fl["synth"] == 8.0 * 64 * 256 * 256 * 257 / 2
    assert fl["factor_gj"] == sum(2.0 * n**3 for n in range(1, 257))
    assert fl["inverse"] > fl["synth"]


def test_cpu_estimate_runs_and_is_positive():
    cfg = dict(bench.CONFIGS[1])
    t, how = bench.cpu_round_trip_estimate(cfg)
    assert t > 0 and "extrapolated" in how


def test_ncu_traffic_reads_committed_profile():
    traffic, src = bench.ncu_traffic("sweep", 256, 64)
    assert traffic is None or (traffic > 1e8 and src.startswith("profiles/"))
