"""Grid input contract of the hot path: ring co-latitudes and grid files.

Mirrors the parts of optisph.sampling the transforms consume
(pkg/src/optisph/sampling.py): ``ColatitudeGrid`` (46-79), the uniform
candidate set (97-105), the interleaved default ordering (181-208) and the
integer-only ``OPTISPH-GRID v1`` cache file (316-370), which reproduces the
co-latitudes bit-exactly.  Condition-minimised orderings are produced by the
reference's greedy optimiser and shipped as grid files (tests/golden/grids);
the sine / tan^(1/3) measures are outside the north_star path.
"""

from __future__ import annotations

import enum
import zlib
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import BandLimitError, FileFormatError

_GRID_MAGIC = "OPTISPH-GRID v1"


class Measure(enum.Enum):
    UNIFORM = "uniform"
    SINE = "sine"
    TAN_CUBE_ROOT = "tan13"


class Ordering(enum.Enum):
    INTERLEAVED = "interleaved"
    CONDITION_MINIMIZED = "condmin"


@dataclass(frozen=True, eq=False)
class ColatitudeGrid:
    """Ring co-latitudes; ``thetas[k]`` is the ring with 2k+1 samples (sampling.py:46-79)."""

    band_limit: int
    thetas: np.ndarray
    permutation: np.ndarray
    measure: Measure = Measure.UNIFORM
    ordering: Ordering = Ordering.CONDITION_MINIMIZED

    def __post_init__(self):
        L = self.band_limit
        if L < 1:
            raise BandLimitError(f"band limit must be positive, got {L}")
        if len(self.thetas) != L or len(self.permutation) != L:
            raise BandLimitError("grid arrays inconsistent with band limit")
        if sorted(int(p) for p in self.permutation) != list(range(L)):
            raise ValueError("permutation is not a bijection on 0..L-1")
        if not np.all((self.thetas > 0.0) & (self.thetas <= np.pi)):
            raise ValueError("co-latitudes must lie in (0, pi]")
        if len(np.unique(self.thetas)) != L:
            raise ValueError("co-latitudes must be distinct")

    @property
    def sample_count(self) -> int:
        return self.band_limit**2

    def ring_sizes(self) -> np.ndarray:
        return 2 * np.arange(self.band_limit) + 1


@dataclass(frozen=True)
class RingLongitudes:
    ring_index: int
    phis: np.ndarray


def ring_longitudes(k: int) -> RingLongitudes:
    """phi_j = 2 pi j / (2k+1) (sampling.py:90-94)."""
    if k < 0:
        raise ValueError(f"ring index must be non-negative, got {k}")
    n = 2 * k + 1
    return RingLongitudes(ring_index=k, phis=2.0 * np.pi * np.arange(n) / n)


def equiangular_candidates(band_limit: int) -> np.ndarray:
    """pi*(2t+1)/(2L-1), t = 0..L-1; the last candidate is exactly pi (sampling.py:97-105)."""
    if band_limit < 1:
        raise BandLimitError(f"band limit must be positive, got {band_limit}")
    t = np.arange(band_limit)
    return np.pi * ((2 * t + 1) / (2 * band_limit - 1))


def candidates(band_limit: int, measure: Measure = Measure.UNIFORM) -> np.ndarray:
    if measure is not Measure.UNIFORM:
        raise NotImplementedError("only the uniform measure is on the north_star path")
    return equiangular_candidates(band_limit)


def interleaved_permutation(band_limit: int) -> np.ndarray:
    """Pole to ring 0, then alternate the remaining extremes (sampling.py:181-189)."""
    L = band_limit
    perm = np.empty(L, dtype=np.int64)
    perm[0] = L - 1
    for k in range(1, L):
        perm[k] = (k - 1) // 2 if k % 2 else L - 1 - k // 2
    return perm


def interleaved_grid(band_limit: int) -> ColatitudeGrid:
    """The reference's make_grid default (sampling.py:192-208, 281-313)."""
    perm = interleaved_permutation(band_limit)
    return ColatitudeGrid(band_limit, equiangular_candidates(band_limit)[perm], perm,
                          Measure.UNIFORM, Ordering.INTERLEAVED)


def grid_from_permutation(band_limit: int, perm, ordering=Ordering.CONDITION_MINIMIZED) -> ColatitudeGrid:
    perm = np.asarray(perm, dtype=np.int64)
    return ColatitudeGrid(band_limit, equiangular_candidates(band_limit)[perm], perm,
                          Measure.UNIFORM, ordering)


def _payload(grid: ColatitudeGrid) -> str:
    lines = [_GRID_MAGIC, f"L {grid.band_limit}", f"measure {grid.measure.value}",
             f"ordering {grid.ordering.value}"]
    lines.extend(str(int(t)) for t in grid.permutation)
    return "\n".join(lines) + "\n"


def save_grid(grid: ColatitudeGrid, destination) -> None:
    """Integer-only grid file with crc32 trailer (sampling.py:316-331)."""
    payload = _payload(grid)
    crc = zlib.crc32(payload.encode("ascii"))
    Path(destination).write_text(payload + f"crc32 {crc:08x}\n", encoding="ascii")


def load_grid(source) -> ColatitudeGrid:
    """Read an OPTISPH-GRID v1 file and rebuild its co-latitudes bit-exactly (sampling.py:334-370)."""
    text = Path(source).read_text(encoding="ascii")
    lines = text.splitlines()
    if not lines or lines[0] != _GRID_MAGIC:
        raise FileFormatError(f"{source}: missing or unsupported grid header")
    if len(lines) < 5:
        raise FileFormatError(f"{source}: truncated grid file")
    if not lines[-1].startswith("crc32 "):
        raise FileFormatError(f"{source}: missing crc32 trailer")
    payload = "\n".join(lines[:-1]) + "\n"
    expected = int(lines[-1].split()[1], 16)
    actual = zlib.crc32(payload.encode("ascii"))
    if actual != expected:
        raise FileFormatError(
            f"{source}: checksum mismatch (stored {expected:08x}, computed {actual:08x})"
        )
    try:
        band_limit = int(lines[1].split()[1])
        measure = Measure(lines[2].split()[1])
        ordering = Ordering(lines[3].split()[1])
        perm = np.array([int(s) for s in lines[4:-1]], dtype=np.int64)
    except (IndexError, ValueError) as exc:
        raise FileFormatError(f"{source}: malformed grid file: {exc}")
    if len(perm) != band_limit:
        raise FileFormatError(f"{source}: expected {band_limit} permutation lines, found {len(perm)}")
    return ColatitudeGrid(band_limit, candidates(band_limit, measure)[perm], perm, measure, ordering)
