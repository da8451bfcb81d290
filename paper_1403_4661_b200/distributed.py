"""Transforms across GPUs, one process per GPU (torch.distributed).

Three partitions of the reference's loops (pkg/src/optisph/transform.py):

* ``sharded_apply`` -- maps: a batch is split into contiguous shards, every
  rank transforms its own maps, no exchange on the data path (weak scaling).
* ``ShardedTransform(mode="factors")`` -- batches without redundant
  factorisation: rank r factors only its block of orders (the per-order
  solves of transform.py:451 are independent and data-free), the factor
  buffers are broadcast from every owner (an all-gather), then each rank
  sweeps its own maps (the L^4/6 factor work is split instead of repeated).
* ``ShardedTransform(mode="chain")`` -- one large map across GPUs.  The
  inverse is split by ring ranges (transform.py:148-201: independent per
  ring) and the ring segments all-gathered.  The forward's order loop
  (transform.py:441-463) is a chain: orders are cut into load-balanced blocks
  descending with the rank (osph_shard_range).  Every rank factors its block
  at once; then rank 0 sweeps its orders and hands the corrected ring spectra
  and the coefficients solved so far to rank 1, which sweeps its block, and so
  on; the last rank broadcasts the completed coefficients.

The data plane is whatever backend the process group uses: NCCL over
NVLink on GPUs (buffers exchanged in place, on the plan's stream = torch's
current stream), or gloo through host memory (used by the CPU-hosted tests:
two ranks may then share one GPU, since no kernel waits on another rank).
Timings are reduced as the max over ranks.
"""

from __future__ import annotations

from typing import Callable

import numpy as np

from . import _lib


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) shard of `total` items for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, group=None) -> float:
    """Max of a scalar over all ranks (timing rule: device time, max over ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sharded_apply(batch: np.ndarray, compute: Callable[[np.ndarray], np.ndarray], group=None,
                  gather: bool = True) -> np.ndarray:
    """Split `batch` (B, L^2) over ranks, run `compute` on the local shard, all-gather.

    `compute` is the per-rank transform (e.g. ``lambda x: inverse_sht_batch(x, grid,
    device=local_rank)``); every rank passes the same full batch.  With
    ``gather=False`` the local shard's result is returned.
    """
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return compute(batch)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_bounds(batch.shape[0], rank, world)
    local = np.ascontiguousarray(compute(batch[lo:hi])) if hi > lo else np.empty((0,) + batch.shape[1:],
                                                                                  batch.dtype)
    if not gather:
        return local
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    width = max(b - a for a, b in (shard_bounds(batch.shape[0], r, world) for r in range(world)))
    buf = torch.zeros((width,) + batch.shape[1:], dtype=torch.complex128, device=dev)
    if hi > lo:
        buf[: hi - lo] = torch.from_numpy(local).to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = []
    for r in range(world):
        a, b = shard_bounds(batch.shape[0], r, world)
        out.append(parts[r][: b - a].cpu().numpy())
    return np.concatenate(out, axis=0)


# ---------------------------------------------------------------------------
# order- and ring-sharded transforms


class _CudaBytes:
    """A raw device range as a __cuda_array_interface__ object (zero-copy torch view)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def device_bytes(ptr: int, nbytes: int, device: int):
    """uint8 torch tensor viewing `nbytes` at device address `ptr` (a plan buffer)."""
    import torch

    return torch.as_tensor(_CudaBytes(ptr, nbytes), device=torch.device("cuda", device))


def shard_range(L: int, rank: int, world: int, mode: int) -> tuple[int, int, int, int]:
    """(m_lo, m_hi, k_lo, k_hi) of `rank` (osph_shard_range): orders [m_lo, m_hi]
    (inclusive), rings [k_lo, k_hi)."""
    import ctypes

    v = [ctypes.c_int() for _ in range(4)]
    lib = _lib.load()
    _lib.raise_for(lib.osph_shard_range(int(L), int(rank), int(world), int(mode), *[ctypes.byref(x) for x in v]))
    return tuple(int(x.value) for x in v)


class ShardedTransform:
    """A grid's transforms on this rank's GPU as one shard of a process group.

    mode="chain":   one map (or a few) across the ranks; every rank passes the
                    same input and gets the full output.
    mode="factors": batches; every rank passes ITS OWN maps; the per-order
                    factorisation is split over the ranks and all-gathered.
    """

    FACTOR_BUFFERS = (_lib.BUF_XT, _lib.BUF_PB, _lib.BUF_AT, _lib.BUF_U, _lib.BUF_W, _lib.BUF_BETA,
                      _lib.BUF_JSTAR, _lib.BUF_NORMS, _lib.BUF_STATUS, _lib.BUF_UT)

    def __init__(self, grid, max_batch: int = 1, mode: str = "chain", group=None, device: int | None = None,
                 plan=None):
        """`plan` (tests only): an object with the Plan methods used below whose
        buffers live in host memory; `device` is then "cpu"."""
        import torch
        import torch.distributed as dist

        from .transform import Plan

        if mode not in ("chain", "factors"):
            raise ValueError(f"unknown shard mode {mode!r}")
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.mode = mode
        self.cmode = _lib.SHARD_CHAIN if mode == "chain" else _lib.SHARD_FACTORS
        self.cuda = device != "cpu"
        self.device = device if not self.cuda else torch.cuda.current_device() if device is None else int(device)
        self.grid = grid
        self.L = grid.band_limit if hasattr(grid, "band_limit") else len(grid)
        thetas = getattr(grid, "thetas", grid)
        self.plan = Plan(thetas, max_batch, self.device) if plan is None else plan
        self.plan.shard(self.rank, self.world, self.cmode)
        self.ranges = [shard_range(self.L, r, self.world, self.cmode) for r in range(self.world)]
        self.nccl = dist.is_initialized() and dist.get_backend(group) == "nccl"

    # -- data plane ---------------------------------------------------------
    def _sync_stream(self):
        import torch

        if self.cuda:
            self.plan.set_stream(_torch_stream(torch.cuda.current_stream(self.device)))

    def _synchronize(self):
        import torch

        if self.cuda:
            torch.cuda.synchronize(self.device)

    def _view(self, ptr: int, nbytes: int):
        """uint8 tensor over a plan buffer (device memory; host memory for a test plan)."""
        import ctypes

        import torch

        if self.cuda:
            return device_bytes(ptr, nbytes, self.device)
        return torch.frombuffer((ctypes.c_uint8 * nbytes).from_address(ptr), dtype=torch.uint8)

    def _bcast(self, view, src: int):
        """Broadcast a device byte view from rank `src` (NCCL in place; gloo via host)."""
        import torch
        import torch.distributed as dist

        if self.world == 1 or view.numel() == 0:
            return
        if self.nccl:
            dist.broadcast(view, src=src, group=self.group)
            return
        self._synchronize()
        host = view.cpu() if self.rank == src else torch.empty(view.numel(), dtype=torch.uint8)
        dist.broadcast(host, src=src, group=self.group)
        if self.rank != src:
            view.copy_(host.to(view.device))

    def _send(self, view, dst: int):
        import torch
        import torch.distributed as dist

        if self.nccl:
            dist.send(view, dst=dst, group=self.group)
        else:
            self._synchronize()
            dist.send(view.cpu(), dst=dst, group=self.group)

    def _recv(self, view, src: int):
        import torch
        import torch.distributed as dist

        if self.nccl:
            dist.recv(view, src=src, group=self.group)
        else:
            host = torch.empty(view.numel(), dtype=torch.uint8)
            dist.recv(host, src=src, group=self.group)
            view.copy_(host.to(view.device))

    # -- transforms ---------------------------------------------------------
    def inverse(self, flm):
        """Samples of the maps (B, L^2) device tensor `flm`.

        chain: rings split over the ranks, every rank returns every ring;
        factors: this rank's own maps."""
        import torch

        x = flm.reshape(-1, self.L * self.L).contiguous()
        B = x.shape[0]
        out = torch.empty_like(x)
        self._sync_stream()
        self.plan.inverse_raw(B, x.data_ptr(), out.data_ptr(), _lib.OSPH_DEVICE | _lib.OSPH_ASYNC)
        if self.mode == "chain" and self.world > 1:
            flat = out.view(torch.uint8).reshape(B, -1)
            for r, (_, _, k_lo, k_hi) in enumerate(self.ranges):
                seg = flat[:, 16 * k_lo * k_lo:16 * k_hi * k_hi]
                tmp = seg.contiguous() if self.rank == r else torch.empty_like(seg)
                self._bcast(tmp.reshape(-1), r)
                if self.rank != r:
                    seg.copy_(tmp)
        return out

    def forward(self, samples, check: bool = False):
        """Coefficients of the maps (B, L^2) device tensor `samples` (see the class docstring)."""
        import torch

        x = samples.reshape(-1, self.L * self.L).contiguous()
        B = x.shape[0]
        self._sync_stream()
        plan = self.plan
        if self.mode == "factors":
            flm = torch.empty_like(x)
            plan.forward_stage(_lib.STAGE_FACTOR, B, 0, 0, _lib.OSPH_DEVICE | _lib.OSPH_ASYNC)
            for q, (m_lo, m_hi, _, _) in enumerate(self.ranges):
                for which in self.FACTOR_BUFFERS:
                    ptr, nbytes = plan.buffer(which, 0, m_lo, m_hi)
                    if nbytes:
                        self._bcast(self._view(ptr, nbytes), q)
            plan.forward_stage(_lib.STAGE_RINGS | _lib.STAGE_SWEEP, B, x.data_ptr(), flm.data_ptr(),
                               _lib.OSPH_DEVICE if check else _lib.OSPH_DEVICE | _lib.OSPH_ASYNC, check)
            return flm
        # chain: rank 0 transforms the rings, every rank factors its block
        flm = torch.zeros_like(x)
        first = _lib.STAGE_RINGS | _lib.STAGE_FACTOR if self.rank == 0 else _lib.STAGE_FACTOR
        plan.forward_stage(first, B, x.data_ptr(), flm.data_ptr(), _lib.OSPH_DEVICE | _lib.OSPH_ASYNC)
        sp_ptr, sp_bytes = plan.buffer(_lib.BUF_SPECTRA, B)
        spectra = self._view(sp_ptr, sp_bytes)
        coeffs = flm.view(torch.uint8).reshape(-1)
        if self.rank > 0:  # spectra corrected by every higher order + the coefficients solved so far
            self._recv(spectra, self.rank - 1)
            self._recv(coeffs, self.rank - 1)
        plan.forward_stage(_lib.STAGE_SWEEP, B, x.data_ptr(), flm.data_ptr(),
                           _lib.OSPH_DEVICE if check else _lib.OSPH_DEVICE | _lib.OSPH_ASYNC, check)
        if self.rank + 1 < self.world:
            self._send(spectra, self.rank + 1)
            self._send(coeffs, self.rank + 1)
        self._bcast(coeffs, self.world - 1)  # the last block completes every order
        return flm

    def close(self):
        self.plan.close()


def _torch_stream(stream) -> int:
    h = int(stream.cuda_stream)
    return h if h != 0 else 1
