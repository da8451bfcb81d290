"""Forward and inverse SHT on the L^2-sample grid -- host side of the B200 path.

Drop-in mirror of the reference's public transform API
(pkg/src/optisph/transform.py): ``HarmonicCoefficients`` (34-68),
``SpatialSamples`` (71-103), ``TransformStats`` (106-112), ``ring_analysis``
(115-131), ``inverse_sht`` (347-357) and ``forward_sht`` (360-393), with the
same signatures, data layouts and exceptions.  Every transform runs in
libosph.so (hand-written sm_100a CUDA) through the C ABI of include/osph.h;
there is no CPU fallback.

Batched entry points ``inverse_sht_batch`` / ``forward_sht_batch`` take
arrays of shape (B, L^2) -- numpy (host memory, copied in/out by the library)
or CUDA torch tensors (device memory, no copies).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import AliasingError, BandLimitError, OrderRangeError

TWO_PI = 2.0 * np.pi


@dataclass
class HarmonicCoefficients:
    """Triangular coefficient storage, flattened as index(ell, m) = ell^2 + ell + m."""

    band_limit: int
    values: np.ndarray

    @staticmethod
    def index(ell: int, m: int) -> int:
        return ell * ell + ell + m

    @classmethod
    def zeros(cls, band_limit: int) -> "HarmonicCoefficients":
        if band_limit < 1:
            raise BandLimitError(f"band limit must be positive, got {band_limit}")
        return cls(band_limit, np.zeros(band_limit**2, dtype=np.complex128))

    def get(self, ell: int, m: int) -> complex:
        return self.values[self.index(ell, m)]

    def set(self, ell: int, m: int, value: complex) -> None:
        self.values[self.index(ell, m)] = value

    def order_slice(self, m: int, ell_min: int | None = None) -> np.ndarray:
        lo = abs(m) if ell_min is None else ell_min
        ells = np.arange(lo, self.band_limit)
        return self.values[ells * ells + ells + m]

    def set_order_slice(self, m: int, values, ell_min: int | None = None) -> None:
        lo = abs(m) if ell_min is None else ell_min
        ells = np.arange(lo, self.band_limit)
        self.values[ells * ells + ells + m] = values

    def copy(self) -> "HarmonicCoefficients":
        return HarmonicCoefficients(self.band_limit, self.values.copy())


@dataclass
class SpatialSamples:
    """Ragged ring storage: ring k holds 2k+1 complex samples."""

    band_limit: int
    rings: list

    @classmethod
    def zeros(cls, band_limit: int) -> "SpatialSamples":
        if band_limit < 1:
            raise BandLimitError(f"band limit must be positive, got {band_limit}")
        return cls(band_limit, [np.zeros(2 * k + 1, dtype=np.complex128) for k in range(band_limit)])

    @classmethod
    def from_flat(cls, band_limit: int, flat) -> "SpatialSamples":
        flat = np.asarray(flat, dtype=np.complex128)
        if flat.size != band_limit**2:
            raise BandLimitError(f"expected {band_limit**2} samples, got {flat.size}")
        return cls(band_limit, [flat[k * k : (k + 1) * (k + 1)].copy() for k in range(band_limit)])

    def flatten(self) -> np.ndarray:
        return np.concatenate(self.rings)

    def copy(self) -> "SpatialSamples":
        return SpatialSamples(self.band_limit, [r.copy() for r in self.rings])

    @property
    def sample_count(self) -> int:
        return sum(len(r) for r in self.rings)


@dataclass
class TransformStats:
    """Timing bookkeeping filled in by ``forward_sht`` (device time, seconds)."""

    solve_seconds: float = 0.0
    orders: int = 0
    extra: dict = field(default_factory=dict)


def _check_band_limits(a: int, b: int) -> None:
    if a != b:
        raise BandLimitError(f"band limits disagree: {a} vs {b}")


# ---------------------------------------------------------------------------
# plans


class Plan:
    """One libosph plan: band limit, ring co-latitudes, batch capacity, device(s).

    ``devices`` (a list) makes one plan over several GPUs driven by this
    process (osph_plan_create with ndev > 1; host buffers only): batches are
    split by maps with the factorisation split by order blocks, single maps
    run as an order-block chain (shard.cu)."""

    def __init__(self, thetas, max_batch: int = 1, device: int = 0, devices=None):
        lib = _lib.load()
        th = np.ascontiguousarray(np.asarray(thetas, dtype=np.float64))
        self.L = int(th.size)
        self.thetas = th
        self.max_batch = int(max_batch)
        devs = [int(device)] if devices is None else [int(d) for d in devices]
        self.devices = devs
        self.device = devs[0]
        dev_arr = (ctypes.c_int * len(devs))(*devs)
        handle = ctypes.c_void_p()
        rc = lib.osph_plan_create(self.L, th.ctypes.data_as(ctypes.c_void_p), self.max_batch, len(devs),
                                  ctypes.cast(dev_arr, ctypes.c_void_p), ctypes.byref(handle))
        _lib.raise_for(rc)
        self._h = handle
        self._lib = lib
        self.lock = threading.Lock()

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.osph_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: int | None) -> None:
        _lib.raise_for(self._lib.osph_plan_set_stream(self._h, ctypes.c_void_p(stream_ptr or 0)))

    def last_launch_count(self) -> int:
        return int(self._lib.osph_last_launch_count(self._h))

    # sharded operation (one process per GPU; distributed.py drives the exchange) ----------
    def shard(self, rank: int, nranks: int, mode: int) -> None:
        """Make this plan rank ``rank`` of ``nranks`` (osph_plan_shard; before its first forward)."""
        _lib.raise_for(self._lib.osph_plan_shard(self._h, int(rank), int(nranks), int(mode)))

    def forward_stage(self, stages: int, B: int, src: int, dst: int, kind: int = _lib.OSPH_DEVICE,
                      check: bool = False) -> None:
        st = _lib.OsphStats()
        rc = self._lib.osph_forward_stage(self._h, int(stages), int(B), ctypes.c_void_p(src), ctypes.c_void_p(dst),
                                          int(kind), 1 if check else 0, ctypes.byref(st))
        _lib.raise_for(rc, st)

    def buffer(self, which: int, B: int = 0, m_lo: int = 0, m_hi: int = 0) -> tuple[int, int]:
        """(device address, bytes) of an exchange buffer (osph_shard_buffer)."""
        ptr = ctypes.c_void_p()
        nbytes = ctypes.c_int64()
        _lib.raise_for(self._lib.osph_shard_buffer(self._h, int(which), int(B), int(m_lo), int(m_hi),
                                                   ctypes.byref(ptr), ctypes.byref(nbytes)))
        return int(ptr.value or 0), int(nbytes.value)

    def last_sweep_kind(self) -> str | None:
        """Sweep variant of the last forward call: persistent / gemm / large / windowed."""
        return _lib.SWEEP_KINDS.get(int(self._lib.osph_last_sweep_kind(self._h)))

    def pivots(self) -> tuple[np.ndarray, float]:
        """(perm packed by order, seconds this plan spent discovering it) -- osph_plan_pivots."""
        perm = np.empty(self.L * (self.L + 1) // 2, dtype=np.int32)
        sec = ctypes.c_double()
        _lib.raise_for(self._lib.osph_plan_pivots(self._h, perm.ctypes.data_as(ctypes.c_void_p), ctypes.byref(sec)))
        return perm, float(sec.value)

    def last_stage_times(self) -> np.ndarray:
        """Device seconds: last inverse's 3 stages, then last forward's 3 (osph_last_stage_times)."""
        out = np.zeros(6)
        _lib.raise_for(self._lib.osph_last_stage_times(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    # raw calls -----------------------------------------------------------
    def inverse_raw(self, B: int, src: int, dst: int, kind: int) -> None:
        _lib.raise_for(self._lib.osph_inverse(self._h, B, ctypes.c_void_p(src), ctypes.c_void_p(dst), kind))

    def spin_inverse_raw(self, spin: int, B: int, src: int, dst: int, kind: int) -> None:
        _lib.raise_for(self._lib.osph_spin_inverse(self._h, int(spin), B, ctypes.c_void_p(src), ctypes.c_void_p(dst),
                                                   kind))

    def spin_forward_raw(self, spin: int, B: int, src: int, dst: int, kind: int, check: bool) -> _lib.OsphStats:
        st = _lib.OsphStats()
        rc = self._lib.osph_spin_forward(self._h, int(spin), B, ctypes.c_void_p(src), ctypes.c_void_p(dst), kind,
                                         1 if check else 0, ctypes.byref(st))
        _lib.raise_for(rc, st)
        return st

    def spin_block(self, spin: int, m: int, out_ptr: int, ld: int) -> None:
        """osph_spin_block into a device buffer (degree-major, leading dimension ld >= L)."""
        _lib.raise_for(self._lib.osph_spin_block(self._h, int(spin), int(m), ctypes.c_void_p(out_ptr), int(ld),
                                                 _lib.OSPH_DEVICE))

    def forward_raw(self, B: int, src: int, dst: int, kind: int, check: bool) -> _lib.OsphStats:
        st = _lib.OsphStats()
        rc = self._lib.osph_forward(self._h, B, ctypes.c_void_p(src), ctypes.c_void_p(dst), kind,
                                    1 if check else 0, ctypes.byref(st))
        _lib.raise_for(rc, st)
        return st


_plans: dict = {}
_plans_lock = threading.Lock()


def get_plan(grid_or_thetas, batch: int = 1, device: int = 0) -> Plan:
    """Cached plan for (device, co-latitudes), grown to hold ``batch`` maps."""
    thetas = getattr(grid_or_thetas, "thetas", grid_or_thetas)
    th = np.ascontiguousarray(np.asarray(thetas, dtype=np.float64))
    key = (int(device), th.size, th.tobytes())
    with _plans_lock:
        plan = _plans.get(key)
        if plan is None or plan.max_batch < batch:
            # a smaller cached plan is only dropped from the cache, never closed here:
            # another thread may hold it (between get_plan and its plan.lock, or inside
            # a call); it is destroyed by Plan.__del__ when the last reference goes
            plan = Plan(th, max(batch, plan.max_batch * 2 if plan else batch), device)
            _plans[key] = plan
        return plan


def clear_plans() -> None:
    with _plans_lock:
        for p in _plans.values():
            with p.lock:  # wait for a call in flight on this plan
                p.close()
        _plans.clear()


# ---------------------------------------------------------------------------
# batched entry points


def torch_stream_handle(stream) -> int:
    """cudaStream_t of a torch stream; torch's default stream (handle 0) maps to
    cudaStreamLegacy (1), since NULL means "plan-owned stream" in the C ABI."""
    h = int(stream.cuda_stream)
    return h if h != 0 else 1


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _check_out(out, shape, device=None):
    """The library writes B * L^2 complex128 values through ``out``: refuse anything else."""
    if out is None:
        return
    if device is not None:  # torch tensor on the input's device
        import torch

        if not _is_torch_cuda(out) or out.device != device:
            raise ValueError(f"out must be a CUDA tensor on {device}")
        if out.dtype != torch.complex128 or not out.is_contiguous() or tuple(out.shape) != tuple(shape):
            raise ValueError(f"out must be a contiguous complex128 tensor of shape {tuple(shape)}")
        return
    if not isinstance(out, np.ndarray):
        raise ValueError("out must be a numpy array for host inputs")
    if out.dtype != np.complex128 or not out.flags.c_contiguous or out.shape != tuple(shape) \
            or not out.flags.writeable:
        raise ValueError(f"out must be a writeable C-contiguous complex128 array of shape {tuple(shape)}")


def _run(direction: str, data, grid, out=None, check: bool = True, device: int = 0, real: bool = False,
         spin: int | None = None):
    """Shared driver: numpy (host) or CUDA torch tensor (device) batches of shape (B, L^2).
    ``spin`` not None: the spin-weighted transforms (osph_spin_*)."""
    L = grid.band_limit if hasattr(grid, "band_limit") else len(grid)

    def call(plan, B, src, dst, kind):
        if spin is not None:
            if direction == "inverse":
                plan.spin_inverse_raw(spin, B, src, dst, kind)
                return None
            return plan.spin_forward_raw(spin, B, src, dst, kind, check)
        if direction == "inverse":
            plan.inverse_raw(B, src, dst, kind)
            return None
        return plan.forward_raw(B, src, dst, kind, check)

    if _is_torch_cuda(data):
        import torch

        if data.dtype != torch.complex128:
            raise TypeError("device batches must be torch.complex128")
        x = data.reshape(-1, L * L) if data.dim() == 2 else data.reshape(1, -1)
        if x.shape[1] != L * L:
            raise BandLimitError(f"expected {L * L} values per map, got {x.shape[1]}")
        x = x.contiguous()
        B = x.shape[0]
        dev = x.device.index or 0
        _check_out(out, x.shape, x.device)
        y = out if out is not None else torch.empty_like(x)
        plan = get_plan(grid, B, dev)
        kind = _lib.OSPH_DEVICE | (_lib.OSPH_REAL if real else 0)
        with plan.lock:
            plan.set_stream(torch_stream_handle(torch.cuda.current_stream(x.device)))
            return y, call(plan, B, x.data_ptr(), y.data_ptr(), kind)
    x = np.ascontiguousarray(np.asarray(data, dtype=np.complex128))
    if x.ndim == 1:
        x = x.reshape(1, -1)
    if x.shape[-1] != L * L:
        raise BandLimitError(f"expected {L * L} values per map, got {x.shape[-1]}")
    B = x.shape[0]
    _check_out(out, x.shape)
    y = out if out is not None else np.empty_like(x)
    plan = get_plan(grid, B, device)
    kind = _lib.OSPH_HOST | (_lib.OSPH_REAL if real else 0)
    with plan.lock:
        plan.set_stream(None)
        return y, call(plan, B, x.ctypes.data, y.ctypes.data, kind)


def inverse_sht_batch(flm, grid, out=None, device: int = 0, *, real: bool = False):
    """B maps at once: flm (B, L^2) in l^2+l+m order -> samples (B, L^2), ring-major.

    ``real=True`` declares real-valued maps (f_{l,-m} = (-1)^m conj f_lm): pairs of
    maps run as one complex transform and the samples come back with zero
    imaginary parts (OSPH_REAL).
    """
    return _run("inverse", flm, grid, out=out, device=device, real=real)[0]


def forward_sht_batch(samples, grid, *, check: bool = True, stats: TransformStats | None = None, out=None,
                      device: int = 0, real: bool = False):
    """B maps at once: samples (B, L^2) -> coefficients (B, L^2).

    ``real=True`` declares real-valued samples (imaginary parts are ignored);
    the coefficients come back complete (both signs of m), as the complex path's.
    """
    y, st = _run("forward", samples, grid, out=out, check=check, device=device, real=real)
    if stats is not None and st is not None:
        stats.solve_seconds = st.solve_seconds
        stats.orders = st.orders
        stats.extra.update(factor_seconds=st.factor_seconds, sweep_seconds=st.sweep_seconds,
                           total_seconds=st.total_seconds)
    return y


# ---------------------------------------------------------------------------
# reference-compatible single-map API


def inverse_sht(coeffs: HarmonicCoefficients, grid) -> SpatialSamples:
    """Synthesize the band-limited signal on every grid sample (transform.py:347-357)."""
    L = grid.band_limit
    _check_band_limits(coeffs.band_limit, L)
    flat = inverse_sht_batch(np.asarray(coeffs.values, dtype=np.complex128).reshape(1, -1), grid)[0]
    return SpatialSamples.from_flat(L, flat)


def forward_sht(samples: SpatialSamples, grid, *, method: str = "direct", check: bool = True,
                stats: TransformStats | None = None) -> HarmonicCoefficients:
    """Recover all L^2 coefficients by top-down order peeling (transform.py:360-393).

    ``method`` is validated like the reference; "direct" and "spectral" both
    run the GPU sweep (the reference's two methods agree to 1e-12,
    test_transform.py:133-137).  The caller's samples are never modified.
    """
    L = grid.band_limit
    _check_band_limits(samples.band_limit, L)
    if method not in ("direct", "spectral"):
        raise ValueError(f"unknown method {method!r}")
    flat = samples.flatten().reshape(1, -1)
    values = forward_sht_batch(flat, grid, check=check, stats=stats)[0]
    return HarmonicCoefficients(L, values)


# ---------------------------------------------------------------------------
# spin-weighted transforms (transform.py:474-533, legendre.py:276-306)


def _check_spin(spin: int, L: int) -> int:
    spin = int(spin)
    if abs(spin) >= L:
        raise OrderRangeError(f"spin {spin} invalid for band limit {L}")
    return spin


def spin_inverse_sht_batch(flm, grid, spin: int, out=None, device: int = 0):
    """B maps of spin-weight ``spin``: flm (B, L^2) -> samples (B, L^2) (numpy or CUDA torch).
    Degrees below |spin| are ignored; spin 0 is inverse_sht_batch."""
    spin = _check_spin(spin, grid.band_limit)
    return _run("inverse", flm, grid, out=out, device=device, spin=spin)[0]


def spin_forward_sht_batch(samples, grid, spin: int, *, check: bool = True, stats: TransformStats | None = None,
                           out=None, device: int = 0):
    """B maps of spin-weight ``spin``: samples (B, L^2) -> coefficients (B, L^2);
    degrees below |spin| come back as exact zeros.  The per-order solution
    operators are built on the first call for a spin (stats.extra["factor_seconds"])."""
    spin = _check_spin(spin, grid.band_limit)
    y, st = _run("forward", samples, grid, out=out, check=check, device=device, spin=spin)
    if stats is not None and st is not None:
        stats.solve_seconds = st.solve_seconds
        stats.orders = st.orders
        stats.extra.update(factor_seconds=st.factor_seconds, sweep_seconds=st.sweep_seconds,
                           total_seconds=st.total_seconds)
    return y


def spin_inverse_sht(coeffs: HarmonicCoefficients, grid, spin: int) -> SpatialSamples:
    """Spin-weighted synthesis (transform.py:474-496).  Spin zero takes the scalar
    path bit for bit; coefficients with degree below |spin| are ignored."""
    L = grid.band_limit
    _check_band_limits(coeffs.band_limit, L)
    spin = _check_spin(spin, L)
    if spin == 0:
        return inverse_sht(coeffs, grid)
    flat = spin_inverse_sht_batch(np.asarray(coeffs.values, dtype=np.complex128).reshape(1, -1), grid, spin)[0]
    return SpatialSamples.from_flat(L, flat)


def spin_forward_sht(samples: SpatialSamples, grid, spin: int, *, check: bool = True) -> HarmonicCoefficients:
    """Spin-weighted analysis by the same top-down peeling (transform.py:499-533);
    tall least-squares blocks for |m| < |spin|; degrees below |spin| come back zero."""
    L = grid.band_limit
    _check_band_limits(samples.band_limit, L)
    spin = _check_spin(spin, L)
    if spin == 0:
        return forward_sht(samples, grid, check=check)
    values = spin_forward_sht_batch(samples.flatten().reshape(1, -1), grid, spin, check=check)[0]
    return HarmonicCoefficients(L, values)


def ring_analysis(ring_values, m: int):
    """Quadrature-exact Fourier pair of one ring at frequencies (+m, -m) (transform.py:115-131)."""
    values = np.ascontiguousarray(np.asarray(ring_values, dtype=np.complex128))
    n = values.shape[0]
    if n % 2 == 0:
        raise ValueError(f"ring length must be odd, got {n}")
    k = (n - 1) // 2
    if abs(m) > k:
        raise AliasingError(f"frequency {m} is not resolvable on a ring of index {k}")
    out = np.empty(4)
    lib = _lib.load()
    rc = lib.osph_ring_analysis(values.ctypes.data_as(ctypes.c_void_p), n, int(m),
                                out.ctypes.data_as(ctypes.c_void_p), 0)
    _lib.raise_for(rc)
    return complex(out[0], out[1]), complex(out[2], out[3])
