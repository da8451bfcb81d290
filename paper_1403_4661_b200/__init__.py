"""B200-native (sm_100a) forward/inverse spherical harmonic transforms on the
optimal-dimensionality L^2-sample grid (Khalid, Kennedy & McEwen, arXiv:1403.4661).

Drop-in for the hot path of the reference package ``optisph``
(pkg/src/optisph/__init__.py:39-48): same names, signatures, layouts
(l^2+l+m coefficients, ring-major samples) and exceptions.  All transform
arithmetic runs in libosph.so (hand-written CUDA, C ABI in include/osph.h).
"""

from .errors import (
    AliasingError,
    BandLimitError,
    DeviceError,
    FileFormatError,
    IllConditionedSolveError,
    OptisphError,
    OrderRangeError,
)
from .sampling import (
    ColatitudeGrid,
    Measure,
    Ordering,
    RingLongitudes,
    candidates,
    equiangular_candidates,
    grid_from_permutation,
    interleaved_grid,
    load_grid,
    ring_longitudes,
    save_grid,
)
from .transform import (
    HarmonicCoefficients,
    Plan,
    SpatialSamples,
    TransformStats,
    clear_plans,
    forward_sht,
    forward_sht_batch,
    get_plan,
    inverse_sht,
    inverse_sht_batch,
    ring_analysis,
    spin_forward_sht,
    spin_forward_sht_batch,
    spin_inverse_sht,
    spin_inverse_sht_batch,
)
from .legendre import LegendreColumn, SpinColumn, legendre_column, legendre_table, spin_column, spin_table
from .blocks import (
    CoefficientSlice,
    GVector,
    LegendreBlock,
    block_for_thetas,
    build_block,
    condition_number,
    solve,
)

from . import distributed, experiments, fileio  # noqa: E402
from .fileio import read_coefficients, read_signal, write_coefficients, write_signal  # noqa: E402
from .gridopt import make_grid  # noqa: E402
from .gridopt import optimize_order_like_reference as optimize_order  # noqa: E402

__all__ = [
    "distributed", "experiments", "fileio", "make_grid", "optimize_order", "read_coefficients", "read_signal", "write_coefficients",
    "write_signal",
    "AliasingError", "BandLimitError", "ColatitudeGrid", "DeviceError", "FileFormatError",
    "HarmonicCoefficients", "IllConditionedSolveError", "Measure", "OptisphError", "Ordering",
    "OrderRangeError", "Plan", "RingLongitudes", "SpatialSamples", "TransformStats", "candidates",
    "clear_plans", "equiangular_candidates", "forward_sht", "forward_sht_batch", "get_plan",
    "grid_from_permutation", "interleaved_grid", "inverse_sht", "inverse_sht_batch", "load_grid",
    "ring_analysis", "ring_longitudes", "save_grid", "spin_forward_sht", "spin_forward_sht_batch",
    "spin_inverse_sht", "spin_inverse_sht_batch", "spin_table", "spin_column", "SpinColumn", "legendre_table",
    "legendre_column", "LegendreColumn", "LegendreBlock", "GVector", "CoefficientSlice", "block_for_thetas",
    "build_block", "condition_number", "solve",
]

__version__ = "0.1.0"
