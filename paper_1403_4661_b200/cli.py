"""Command-line front end for the transform path (the reference's cli.py:138-157, 244-253).

    python -m paper_1403_4661_b200.cli grid -L 2048 -o grid.txt [--ordering condmin|interleaved]
    python -m paper_1403_4661_b200.cli forward --signal s.txt --grid grid.txt -o coeffs.txt
    python -m paper_1403_4661_b200.cli inverse --coeffs c.txt --grid grid.txt -o signal.txt

Same file formats (fileio.py) and exit codes as the reference: 0 success,
1 numeric failure (e.g. IllConditionedSolveError), 2 usage or parse failure
(BandLimitError, FileFormatError, bad arguments).  ``grid`` runs the
condition-minimising greedy on the GPU (gridopt.py).  The reference's
``--oracle`` (dense least squares) and experiment subcommands are outside
this package's scope.
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
    return parser


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


_COMMANDS = {"grid": cmd_grid, "forward": cmd_forward, "inverse": cmd_inverse}


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
