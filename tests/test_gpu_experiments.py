"""GPU experiment harness against the reference's own reports.

tests/golden/experiments/*.csv were written by the reference CLI
(tests/golden/make_golden_experiments.py).  The same commands run here
through paper_1403_4661_b200.cli on the B200: same provenance line, header,
rows and keys; error columns within the north_star bar (both sides are
rounding-level, ~1e-15); condition numbers equal to SVD rounding.
"""

import csv
import math
from pathlib import Path

import pytest

from paper_1403_4661_b200.cli import main

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "experiments"
COMMANDS = {
    "exp1.csv": ["exp1", "-L", "8,16,32", "--trials", "3", "--seed", "5"],
    "exp2.csv": ["exp2", "-L", "8,16,32", "--trials", "3", "--seed", "6"],
    "errsurface.csv": ["errsurface", "-L", "16", "--trials", "2", "--seed", "7"],
    "cond_interleaved.csv": ["cond", "-L", "16,32"],
    "cond_condmin.csv": ["cond", "-L", "16,32", "--ordering", "condmin"],
}


def read(path):
    lines = Path(path).read_text().splitlines()
    return lines[0], list(csv.DictReader(lines[1:]))


@pytest.mark.parametrize("name", sorted(COMMANDS))
def test_report_matches_reference(name, tmp_path):
    out = tmp_path / name
    assert main(COMMANDS[name] + ["-o", str(out)]) == 0
    head_ref, rows_ref = read(GOLD / name)
    head, rows = read(out)
    assert head == head_ref
    assert len(rows) == len(rows_ref)
    for r, q in zip(rows, rows_ref):
        assert r.keys() == q.keys()
        for k in r:
            if k in ("L", "trials", "ell", "m"):
                assert r[k] == q[k]
            elif k == "kappa":
                assert math.isclose(float(r[k]), float(q[k]), rel_tol=1e-9), (r, q)
            else:  # round-trip errors: rounding level on both sides
                assert float(r[k]) <= max(1e-11, 10 * float(q[k])), (k, r, q)


def test_bench_report(tmp_path):
    out = tmp_path / "bench.csv"
    assert main(["bench", "-L", "32,64", "--trials", "2", "-o", str(out)]) == 0
    head, rows = read(out)
    assert head == "# optisph bench seed=0"
    assert [r["L"] for r in rows] == ["32", "64"]
    for r in rows:
        assert float(r["tau_i"]) > 0 and float(r["tau_f"]) > 0 and float(r["tau_f1"]) > 0


def test_exp1_large_band_limit(tmp_path):
    """The point of a GPU harness: E1 at L=512 (reference: minutes per trial) in seconds."""
    from paper_1403_4661_b200 import experiments, sampling

    cfg = experiments.SweepConfig(band_limits=(512,), trials=4, seed=1,
                                  cache_dir=str(Path(__file__).resolve().parent / "golden" / "grids"))
    rows = experiments.run_spectral_experiment(cfg)
    assert rows[0]["L"] == 512 and rows[0]["e_max"] < 1e-9
    assert sampling.Ordering.CONDITION_MINIMIZED is cfg.ordering
