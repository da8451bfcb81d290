"""File formats and CLI (fileio.py, cli.py) against files written by the reference's fileio."""

import subprocess
import sys

import numpy as np
import pytest

import paper_1403_4661_b200 as osp
from paper_1403_4661_b200 import cli, fileio
from paper_1403_4661_b200.errors import FileFormatError

from conftest import GOLDEN, GRIDS, ROOT

FIO = GOLDEN / "fileio"


def test_writers_match_reference_bytes(tmp_path):
    v = np.load(FIO / "values_L4.npz")
    fileio.write_coefficients(tmp_path / "c.txt", osp.HarmonicCoefficients(4, v["flm"]))
    fileio.write_signal(tmp_path / "s.txt", osp.SpatialSamples.from_flat(4, v["samples"]))
    assert (tmp_path / "c.txt").read_bytes() == (FIO / "coef_L4.txt").read_bytes()
    assert (tmp_path / "s.txt").read_bytes() == (FIO / "sig_L4.txt").read_bytes()


def test_readers_parse_reference_files():
    v = np.load(FIO / "values_L4.npz")
    c = fileio.read_coefficients(FIO / "coef_L4.txt")
    s = fileio.read_signal(FIO / "sig_L4.txt")
    assert c.band_limit == 4 and np.array_equal(c.values, v["flm"])
    assert np.array_equal(s.flatten(), v["samples"])


@pytest.mark.parametrize("mutate", ["header", "count", "sequence", "fields"])
def test_malformed_files_raise(tmp_path, mutate):
    lines = (FIO / "coef_L4.txt").read_text().splitlines()
    if mutate == "header":
        lines[0] = "OPTISPH-COEF v2"
    elif mutate == "count":
        lines = lines[:-1]
    elif mutate == "sequence":
        lines[3], lines[4] = lines[4], lines[3]
    else:
        lines[5] = "1 0 0.5"
    (tmp_path / "bad.txt").write_text("\n".join(lines) + "\n")
    with pytest.raises(FileFormatError):
        fileio.read_coefficients(tmp_path / "bad.txt")


def test_cli_usage_errors_exit_2(tmp_path, capsys):
    # malformed input: parse failure before any device work
    (tmp_path / "bad.txt").write_text("garbage\n")
    assert cli.main(["forward", "--signal", str(tmp_path / "bad.txt"), "--grid",
                     str(GRIDS / "grid-L8-uniform-condmin.txt"), "-o", str(tmp_path / "o.txt")]) == 2
    # band-limit mismatch between the file (L=4) and the grid (L=8)
    assert cli.main(["inverse", "--coeffs", str(FIO / "coef_L4.txt"), "--grid",
                     str(GRIDS / "grid-L8-uniform-condmin.txt"), "-o", str(tmp_path / "o.txt")]) == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["forward", "--signal", "x"])
    assert e.value.code == 2


@pytest.mark.gpu
def test_cli_round_trip_on_gpu(tmp_path):
    L = 8
    rng = np.random.default_rng(8)
    f = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
    fileio.write_coefficients(tmp_path / "c.txt", osp.HarmonicCoefficients(L, f))
    grid = str(GRIDS / "grid-L8-uniform-condmin.txt")
    run = [sys.executable, "-m", "paper_1403_4661_b200.cli"]
    assert subprocess.run(run + ["inverse", "--coeffs", str(tmp_path / "c.txt"), "--grid", grid,
                                 "-o", str(tmp_path / "s.txt")], cwd=ROOT).returncode == 0
    assert subprocess.run(run + ["forward", "--signal", str(tmp_path / "s.txt"), "--grid", grid,
                                 "-o", str(tmp_path / "c2.txt")], cwd=ROOT).returncode == 0
    back = fileio.read_coefficients(tmp_path / "c2.txt").values
    assert np.abs(back - f).max() <= 1e-12
    # the grid subcommand reproduces the committed (reference-made) grid file
    assert subprocess.run(run + ["grid", "-L", "16", "-o", str(tmp_path / "g.txt")], cwd=ROOT).returncode == 0
    assert np.array_equal(osp.load_grid(tmp_path / "g.txt").permutation,
                          osp.load_grid(GRIDS / "grid-L16-uniform-condmin.txt").permutation)
