"""ctypes binding of libosph.so (include/osph.h).

This is the reference-side binding a maintainer would add.
There is no fallback: if the shared library is missing or no CUDA device is
present, the calls raise.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import BandLimitError, DeviceError, IllConditionedSolveError, OrderRangeError

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libosph.so"

OSPH_OK, OSPH_ERR_ARG, OSPH_ERR_ILLCOND, OSPH_ERR_CUDA, OSPH_ERR_NCCL, OSPH_ERR_ORDER = 0, 1, 2, 3, 4, 5
OSPH_HOST, OSPH_DEVICE, OSPH_ASYNC, OSPH_REAL = 0, 1, 2, 4
SHARD_CHAIN, SHARD_FACTORS = 1, 2
STAGE_RINGS, STAGE_FACTOR, STAGE_SWEEP = 1, 2, 4
BUF_SPECTRA, BUF_XT, BUF_PB, BUF_AT, BUF_U, BUF_W, BUF_BETA, BUF_JSTAR, BUF_NORMS, BUF_STATUS, BUF_UT, BUF_COUNT = range(12)
SWEEP_KINDS = {0: "persistent", 1: "gemm", 2: "large", 3: "windowed", 4: "blocked"}
ABI_VERSION = 3


class OsphStats(ctypes.Structure):
    _fields_ = [
        ("solve_seconds", ctypes.c_double),
        ("orders", ctypes.c_int32),
        ("failed_order", ctypes.c_int32),
        ("failed_kappa", ctypes.c_double),
        ("factor_seconds", ctypes.c_double),
        ("sweep_seconds", ctypes.c_double),
        ("total_seconds", ctypes.c_double),
    ]


# every symbol include/osph.h declares, with (restype, argtypes)
_P = ctypes.c_void_p
_I = ctypes.c_int
SIGNATURES = {
    "osph_plan_create": (_I, [_I, _P, _I, _I, _P, ctypes.POINTER(_P)]),
    "osph_plan_shard": (_I, [_P, _I, _I, _I]),
    "osph_shard_range": (_I, [_I, _I, _I, _I, _P, _P, _P, _P]),
    "osph_forward_stage": (_I, [_P, _I, _I, _P, _P, _I, _I, ctypes.POINTER(OsphStats)]),
    "osph_shard_buffer": (_I, [_P, _I, _I, _I, _I, ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_int64)]),
    "osph_plan_destroy": (_I, [_P]),
    "osph_plan_set_stream": (_I, [_P, _P]),
    "osph_plan_info": (_I, [_P, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "osph_inverse": (_I, [_P, _I, _P, _P, _I]),
    "osph_forward": (_I, [_P, _I, _P, _P, _I, _I, ctypes.POINTER(OsphStats)]),
    "osph_ring_analysis": (_I, [_P, _I, _I, _P, _I]),
    "osph_legendre_block": (_I, [_P, _I, _P, ctypes.c_int64, _I]),
    "osph_last_launch_count": (_I, [_P]),
    "osph_last_sweep_kind": (_I, [_P]),
    "osph_plan_pivots": (_I, [_P, _P, _P]),
    "osph_last_stage_times": (_I, [_P, _P]),
    "osph_spin_inverse": (_I, [_P, _I, _I, _P, _P, _I]),
    "osph_spin_forward": (_I, [_P, _I, _I, _P, _P, _I, _I, ctypes.POINTER(OsphStats)]),
    "osph_spin_block": (_I, [_P, _I, _I, _P, ctypes.c_int64, _I]),
    "osph_spin_seed": (_I, [_I, _I, ctypes.POINTER(_I), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I),
                            ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "osph_last_error": (ctypes.c_char_p, []),
    "osph_abi_version": (_I, []),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libosph.so once; raise if it is absent (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("OSPH_LIB", LIB_PATH))
    if not path.exists():
        raise DeviceError(
            f"{path} not found: build it with `python -m paper_1403_4661_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.osph_abi_version() != ABI_VERSION:
        raise DeviceError(f"{path}: ABI version {lib.osph_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def last_error() -> str:
    return load().osph_last_error().decode("utf-8", "replace")


def raise_for(rc: int, stats: OsphStats | None = None) -> None:
    """Map OSPH_* codes onto the reference's exception types."""
    if rc == OSPH_OK:
        return
    msg = last_error()
    if rc == OSPH_ERR_ILLCOND:
        order = stats.failed_order if stats is not None else -1
        kappa = stats.failed_kappa if stats is not None else float("inf")
        raise IllConditionedSolveError(order, kappa)
    if rc == OSPH_ERR_ARG:
        raise BandLimitError(msg) if "band" in msg or "batch" in msg else ValueError(msg)
    if rc == OSPH_ERR_ORDER:
        raise OrderRangeError(msg)
    if rc == OSPH_ERR_NCCL:
        raise DeviceError(f"libosph multi-GPU exchange failed: {msg}")
    raise DeviceError(f"libosph error {rc}: {msg}")
