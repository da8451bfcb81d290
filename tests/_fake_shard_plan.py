"""A host-memory stand-in for a sharded Plan (tests only).

It keeps the staging contract of osph_forward_stage / osph_shard_buffer /
osph_inverse for a sharded plan (csrc/shard.cu) -- which orders a rank
factors and sweeps, that the ring spectra are corrected by every swept order,
that a chain rank's inverse fills only its own rings -- with trivial
arithmetic in place of the transforms, so ShardedTransform's exchange logic
(who sends which buffer to whom, and when) can run over gloo on CPU.  A
1-rank run is the reference: any missing or misordered exchange changes
the result."""

import ctypes

import numpy as np

from paper_1403_4661_b200 import _lib
from paper_1403_4661_b200.distributed import shard_range


def _array(ptr, n, dtype):
    size = n * np.dtype(dtype).itemsize
    return np.frombuffer((ctypes.c_uint8 * size).from_address(ptr), dtype=dtype)


class FakeShardPlan:
    def __init__(self, L, max_batch):
        self.L, self.max_batch = L, max_batch
        self.spectra = np.zeros((max_batch, L * L), np.complex128)
        self.xt = np.zeros(L, np.float64)
        self.rank, self.world, self.mode = 0, 1, _lib.SHARD_FACTORS
        self.m_lo, self.m_hi, self.k_lo, self.k_hi = 0, L - 1, 0, L  # orders inclusive, rings half-open
        self.stages = []

    def shard(self, rank, world, mode):
        self.rank, self.world, self.mode = rank, world, mode
        self.m_lo, self.m_hi, self.k_lo, self.k_hi = shard_range(self.L, rank, world, mode)

    def set_stream(self, _):
        pass

    def close(self):
        pass

    def buffer(self, which, B=0, m_lo=0, m_hi=0):
        if which == _lib.BUF_SPECTRA:
            return self.spectra.ctypes.data, B * self.L * self.L * 16
        if which == _lib.BUF_XT:
            return self.xt.ctypes.data + 8 * m_lo, 8 * (m_hi - m_lo + 1)
        return 0, 0

    def inverse_raw(self, B, src, dst, kind):
        n = self.L * self.L
        x = _array(src, B * n, np.complex128).reshape(B, n)
        out = _array(dst, B * n, np.complex128).reshape(B, n)
        out[:] = np.nan  # a chain rank computes its own rings only
        a, b = self.k_lo ** 2, self.k_hi ** 2
        out[:, a:b] = 2.0 * x[:, a:b] + (1.0 + 0.5j)

    def forward_stage(self, stages, B, src, dst, kind=0, check=False):
        self.stages.append(stages)
        n = self.L * self.L
        sp = self.spectra[:B]
        if stages & _lib.STAGE_RINGS:
            sp[:] = _array(src, B * n, np.complex128).reshape(B, n)
        if stages & _lib.STAGE_FACTOR:
            for m in range(self.m_lo, self.m_hi + 1):
                self.xt[m] = 1.0 + 0.25 * m
        if stages & _lib.STAGE_SWEEP:
            flm = _array(dst, B * n, np.complex128).reshape(B, n)
            chain = self.mode == _lib.SHARD_CHAIN
            lo, hi = (self.m_lo, self.m_hi) if chain else (0, self.L - 1)
            for m in range(hi, lo - 1, -1):  # descending orders, as the sweep
                # order m "solves" its degrees from the corrected spectra...
                sl = slice(m * self.L, (m + 1) * self.L)
                prev = flm[:, (m + 1) * self.L:(m + 2) * self.L] if m + 1 < self.L else 0.0
                flm[:, sl] = sp[:, sl] * self.xt[m] + 0.125 * prev
                # ...and corrects every lower order's spectra
                sp[:, : m * self.L] += 0.5 * flm[:, sl].sum(axis=1, keepdims=True)
