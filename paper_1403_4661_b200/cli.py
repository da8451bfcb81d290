"""Command-line front end (the reference's cli.py:40-253).

    python -m paper_1403_4661_b200.cli grid -L 2048 -o grid.txt [--ordering condmin|interleaved]
    python -m paper_1403_4661_b200.cli forward --signal s.txt --grid grid.txt -o coeffs.txt
    python -m paper_1403_4661_b200.cli inverse --coeffs c.txt --grid grid.txt -o signal.txt
    python -m paper_1403_4661_b200.cli exp1|exp2 -L 64,128,256 [--trials 10 --seed 0] -o out.csv
    python -m paper_1403_4661_b200.cli errsurface -L 256 -o out.csv
    python -m paper_1403_4661_b200.cli cond -L 64,256 -o out.csv
    python -m paper_1403_4661_b200.cli bench -L 64,128,256 [--trials 3 --mean] -o out.csv

Same file formats (fileio.py), report CSVs (``# optisph <command> seed=<n>``)
and exit codes as the reference: 0 success, 1 numeric failure (e.g.
IllConditionedSolveError), 2 usage or parse failure (BandLimitError,
FileFormatError, bad arguments).  Every transform and the ``grid`` greedy run
on the GPU (experiments.py, gridopt.py).  The reference's ``--oracle`` (dense
least squares / brute-force synthesis, O(L^6) test oracles) and the sine /
tan^(1/3) measures are outside this package's scope (exit 2).
"""

from __future__ import annotations

import argparse
import sys

from . import fileio, sampling
from .errors import BandLimitError, FileFormatError, OptisphError

USAGE_ERRORS = (BandLimitError, FileFormatError)


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse exits 2 on usage errors, as the reference
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        raise SystemExit(2)


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="optisph-b200", description="L^2-sample spherical harmonic transforms on a B200")
    sub = parser.add_subparsers(dest="command", required=True, parser_class=_Parser)
    p = sub.add_parser("grid", help="generate a grid and write its cache file")
    p.add_argument("-L", "--band-limit", type=int, required=True)
    p.add_argument("--ordering", choices=["condmin", "interleaved"], default="condmin")
    p.add_argument("-o", "--out", required=True)
    p = sub.add_parser("forward", help="signal file -> coefficient file")
    p.add_argument("--signal", required=True)
    p.add_argument("--grid", required=True)
    p.add_argument("-o", "--out", required=True)
    p.add_argument("--no-check", action="store_true", help="skip the per-order conditioning check")
    p = sub.add_parser("inverse", help="coefficient file -> signal file")
    p.add_argument("--coeffs", required=True)
    p.add_argument("--grid", required=True)
    p.add_argument("-o", "--out", required=True)
    for name, what in (("exp1", "spectral-spatial-spectral accuracy sweep"),
                       ("exp2", "spatial-spectral-spatial accuracy sweep")):
        p = sub.add_parser(name, help=what)
        p.add_argument("-L", "--band-limits", type=_band_limit_list, required=True)
        p.add_argument("--trials", type=int, default=10)
        p.add_argument("--seed", type=int, default=0)
        _add_grid_options(p)
        p.add_argument("-o", "--out", required=True)
    p = sub.add_parser("errsurface", help="per-(ell, m) round-trip error surface")
    p.add_argument("-L", "--band-limit", type=int, required=True)
    p.add_argument("--trials", type=int, default=10)
    p.add_argument("--seed", type=int, default=0)
    _add_grid_options(p)
    p.add_argument("-o", "--out", required=True)
    p = sub.add_parser("cond", help="per-order condition numbers")
    p.add_argument("-L", "--band-limits", type=_band_limit_list, required=True)
    _add_grid_options(p, default_ordering="interleaved")
    p.add_argument("-o", "--out", required=True)
    p = sub.add_parser("bench", help="transform wall times")
    p.add_argument("-L", "--band-limits", type=_band_limit_list, required=True)
    p.add_argument("--trials", type=int, default=3)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--mean", action="store_true", help="aggregate trials by mean instead of median")
    _add_grid_options(p, default_ordering="interleaved")
    p.add_argument("-o", "--out", required=True)
    return parser


def _band_limit_list(text: str):
    try:
        values = [int(s) for s in text.split(",") if s]
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers, got {text!r}")
    if not values or any(v < 1 for v in values):
        raise argparse.ArgumentTypeError("band limits must be positive integers")
    return tuple(values)


def _add_grid_options(p, default_ordering="condmin"):
    p.add_argument("--measure", choices=["uniform", "sine", "tan13"], default="uniform")
    p.add_argument("--ordering", choices=["interleaved", "condmin"], default=default_ordering)
    p.add_argument("--cache-dir", default=None, help="directory for grid cache files")


def _measure(args):
    if args.measure != "uniform":
        raise BandLimitError(f"measure {args.measure!r} is not supported (uniform only)")
    return sampling.Measure.UNIFORM


def _sweep_config(args):
    from . import experiments

    return experiments.SweepConfig(band_limits=args.band_limits, trials=args.trials, seed=args.seed,
                                   measure=_measure(args), ordering=sampling.Ordering(args.ordering),
                                   cache_dir=args.cache_dir)


def cmd_exp1(args) -> int:
    from . import experiments

    rows = experiments.run_spectral_experiment(_sweep_config(args))
    fileio.write_report(args.out, "exp1", args.seed, ["L", "trials", "e_max", "e_mean"], rows)
    return 0


def cmd_exp2(args) -> int:
    from . import experiments

    rows = experiments.run_spatial_experiment(_sweep_config(args))
    fileio.write_report(args.out, "exp2", args.seed, ["L", "trials", "e_max", "e_mean"], rows)
    return 0


def cmd_errsurface(args) -> int:
    from . import experiments
    from .gridopt import make_grid

    grid = make_grid(args.band_limit, _measure(args), sampling.Ordering(args.ordering), cache_dir=args.cache_dir)
    rows = experiments.error_surface(grid, args.trials, args.seed)
    fileio.write_report(args.out, "errsurface", args.seed, ["ell", "m", "e"], rows)
    return 0


def cmd_cond(args) -> int:
    from . import experiments

    rows = experiments.condition_rows(args.band_limits, _measure(args), sampling.Ordering(args.ordering),
                                      args.cache_dir)
    fileio.write_report(args.out, "cond", 0, ["L", "m", "kappa"], rows)
    finite = [r["kappa"] for r in rows if r["m"] == "max"]
    for L, kemax in zip(args.band_limits, finite):
        print(f"L={L} max_kappa={kemax:.6e}")
    return 0


def cmd_bench(args) -> int:
    from . import experiments

    results = experiments.benchmark(args.band_limits, trials=args.trials, seed=args.seed, measure=_measure(args),
                                    ordering=sampling.Ordering(args.ordering), cache_dir=args.cache_dir,
                                    aggregate="mean" if args.mean else "median")
    rows = [{"L": r.band_limit, "trials": r.trials, "tau_i": r.tau_inverse, "tau_f": r.tau_forward,
             "tau_f1": r.tau_solve} for r in results]
    fileio.write_report(args.out, "bench", args.seed, ["L", "trials", "tau_i", "tau_f", "tau_f1"], rows)
    return 0


def _load_grid_checked(path, expected_L, what):
    grid = sampling.load_grid(path)
    if grid.band_limit != expected_L:
        raise BandLimitError(f"band limit mismatch: {what} has L={expected_L}, grid has L={grid.band_limit}")
    return grid


def cmd_grid(args) -> int:
    if args.band_limit < 1:
        raise BandLimitError(f"band limit must be positive, got {args.band_limit}")
    if args.ordering == "interleaved":
        grid = sampling.interleaved_grid(args.band_limit)
    else:
        from .gridopt import optimize_order

        grid = optimize_order(args.band_limit)
    sampling.save_grid(grid, args.out)
    print(f"grid L={args.band_limit} measure=uniform ordering={args.ordering} samples={args.band_limit ** 2}")
    return 0


def cmd_forward(args) -> int:
    from .transform import forward_sht

    samples = fileio.read_signal(args.signal)
    grid = _load_grid_checked(args.grid, samples.band_limit, args.signal)
    fileio.write_coefficients(args.out, forward_sht(samples, grid, check=not args.no_check))
    return 0


def cmd_inverse(args) -> int:
    from .transform import inverse_sht

    coeffs = fileio.read_coefficients(args.coeffs)
    grid = _load_grid_checked(args.grid, coeffs.band_limit, args.coeffs)
    fileio.write_signal(args.out, inverse_sht(coeffs, grid))
    return 0


_COMMANDS = {"grid": cmd_grid, "forward": cmd_forward, "inverse": cmd_inverse, "exp1": cmd_exp1, "exp2": cmd_exp2,
             "errsurface": cmd_errsurface, "cond": cmd_cond, "bench": cmd_bench}


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return _COMMANDS[args.command](args)
    except USAGE_ERRORS as exc:
        print(f"optisph-b200: {exc}", file=sys.stderr)
        return 2
    except OptisphError as exc:
        print(f"optisph-b200: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
