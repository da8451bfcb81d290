// fft.cuh -- in-shared-memory power-of-two FFT used by the Bluestein ring DFTs.
//
// The reference computes every ring DFT with numpy.fft (pocketfft) at the
// ring's native odd length n = 2k+1 (pkg/src/optisph/transform.py:129, 343,
// 439).  Odd lengths are often prime, so on the GPU each ring DFT is a
// Bluestein chirp-z transform: a length-N (power of two, N >= 2n-1) circular
// convolution computed with two of the FFTs below.
#pragma once
#include "common.cuh"

#define OSPH_TW_SIZE 16384  // twiddle table resolution: tw[j] = e^{-2 pi i j / 16384}, j < 8192

__device__ __forceinline__ double2 tw_load(const double2* __restrict__ tw, int idx, bool inverse) {
  double2 w = __ldg(tw + idx);
  return inverse ? conj2(w) : w;
}

// In-place decimation-in-time FFT of x[0..N) (input already in bit-reversed
// order).  inverse=false: X_q = sum x_t e^{-2 pi i qt/N}; inverse=true uses
// e^{+2 pi i qt/N} and does NOT divide by N.  All threads of the block call it;
// it starts and ends with __syncthreads().
static __device__ void fft_dit_smem(double2* x, int N, int logN, const double2* __restrict__ tw, bool inverse) {
  __syncthreads();
  int h = 1;
  if (logN & 1) {  // one radix-2 stage (span 1, twiddle 1)
    for (int j = threadIdx.x; j < N / 2; j += blockDim.x) {
      double2 a = x[2 * j], b = x[2 * j + 1];
      x[2 * j] = cadd(a, b);
      x[2 * j + 1] = csub(a, b);
    }
    h = 2;
    __syncthreads();
  }
  for (; h < N; h *= 4) {
    const int q = N / 4;
    const int s2 = OSPH_TW_SIZE / (2 * h);
    const int s4 = OSPH_TW_SIZE / (4 * h);
    for (int j = threadIdx.x; j < q; j += blockDim.x) {
      const int pos = j & (h - 1);
      const int base = (j - pos) * 4;
      const int i0 = base + pos, i1 = i0 + h, i2 = i1 + h, i3 = i2 + h;
      const double2 w1 = tw_load(tw, pos * s2, inverse);
      const double2 w2 = tw_load(tw, pos * s4, inverse);
      double2 a0 = x[i0], a1 = cmul(w1, x[i1]), a2 = x[i2], a3 = cmul(w1, x[i3]);
      double2 b0 = cadd(a0, a1), b1 = csub(a0, a1), b2 = cadd(a2, a3), b3 = csub(a2, a3);
      double2 c2 = cmul(w2, b2);
      double2 c3 = cmul(w2, b3);
      // w3 = w2 * (-i) forward, w2 * (+i) inverse
      c3 = inverse ? make_double2(-c3.y, c3.x) : make_double2(c3.y, -c3.x);
      x[i0] = cadd(b0, c2);
      x[i2] = csub(b0, c2);
      x[i1] = cadd(b1, c3);
      x[i3] = csub(b1, c3);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int bitrev(int t, int logN) { return (int)(__brev((unsigned)t) >> (32 - logN)); }

// G independent transforms of length N stored back to back (x[g*N + t]), all
// in bit-reversed order on entry; one pass per radix-4 stage over all G, so
// the stage barriers are shared by the batch.
// twn: shared-memory table e^{-2 pi i j / N}, j < N/2 (see load_twiddles).
static __device__ void fft_dit_smem_multi(double2* x, int N, int logN, int G, const double2* twn, bool inverse) {
  __syncthreads();
  int lh = 0;  // log2 of the current span h
  if (logN & 1) {
    const int half = N >> 1;
    for (int j = threadIdx.x; j < G * half; j += blockDim.x) {
      double2* xg = x + (j >> (logN - 1)) * N;
      const int jj = j & (half - 1);
      double2 a = xg[2 * jj], b = xg[2 * jj + 1];
      xg[2 * jj] = cadd(a, b);
      xg[2 * jj + 1] = csub(a, b);
    }
    lh = 1;
    __syncthreads();
  }
  const int lq = logN - 2;  // log2(N/4)
  for (; lh < logN; lh += 2) {
    const int h = 1 << lh;
    const int sh2 = logN - (lh + 1), sh4 = logN - (lh + 2);
    for (int j = threadIdx.x; j < (G << lq); j += blockDim.x) {
      double2* xg = x + (j >> lq) * N;
      const int jj = j & ((1 << lq) - 1);
      const int pos = jj & (h - 1);
      const int i0 = ((jj - pos) << 2) + pos, i1 = i0 + h, i2 = i1 + h, i3 = i2 + h;
      double2 w1 = twn[pos << sh2], w2 = twn[pos << sh4];
      if (inverse) {
        w1 = conj2(w1);
        w2 = conj2(w2);
      }
      double2 a0 = xg[i0], a1 = cmul(w1, xg[i1]), a2 = xg[i2], a3 = cmul(w1, xg[i3]);
      double2 b0 = cadd(a0, a1), b1 = csub(a0, a1), b2 = cadd(a2, a3), b3 = csub(a2, a3);
      double2 c2 = cmul(w2, b2);
      double2 c3 = cmul(w2, b3);
      c3 = inverse ? make_double2(-c3.y, c3.x) : make_double2(c3.y, -c3.x);
      xg[i0] = cadd(b0, c2);
      xg[i2] = csub(b0, c2);
      xg[i1] = cadd(b1, c3);
      xg[i3] = csub(b1, c3);
    }
    __syncthreads();
  }
}

// twn[j] = e^{-2 pi i j / N}, j < N/2, from the global OSPH_TW_SIZE table (N <= OSPH_TW_SIZE).
__device__ __forceinline__ void load_twiddles(double2* twn, int logN, const double2* __restrict__ tw) {
  const int half = 1 << (logN - 1);
  const int sh = 14 - logN;
  for (int j = threadIdx.x; j < half; j += blockDim.x) twn[j] = __ldg(tw + (j << sh));
}

// ---------------------------------------------------------------------------
// Bluestein convolution pair without bit-reversal passes: forward transform by
// decimation in FREQUENCY (natural order in, bit-reversed out), pointwise
// product with a kernel spectrum stored in bit-reversed order, inverse
// transform by decimation in TIME (bit-reversed in, natural out).  Shared
// memory is addressed through the swizzle fsw(e) = e ^ ((e >> 2) & 7), which
// keeps the strided butterflies of the short-span stages bank-conflict free
// (16-byte elements, N >= 32).

__device__ __forceinline__ int fsw(int e) { return e ^ ((e >> 2) & 7); }

// Per-stage twiddles (layout: see load_stage_twiddles).  The entries of the
// short spans (h < 1024, the first OSPH_SW_SMEM) are copied to shared memory;
// the few long-span stages read the plan's global table (L1/L2 resident), so
// an 8192-point transform fits one CTA next to its data.
struct StageTw {
  const double2* s;
  const double2* __restrict__ g;
  __device__ __forceinline__ double2 operator()(int i) const { return i < OSPH_SW_SMEM ? s[i] : __ldg(g + i); }
};

// smem copy of the first min(N, OSPH_SW_SMEM) entries of the global stage table
__device__ __forceinline__ void load_stage_twiddles_smem(double2* sw, int logN, const double2* __restrict__ gsw) {
  const int cnt = min(1 << logN, OSPH_SW_SMEM);
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) sw[j] = __ldg(gsw + j);
}

// forward-sign DIF, G transforms of length N (x[g*N + fsw(t)])
static __device__ void fft_dif_fwd_multi(double2* x, int logN, int G, const StageTw twn) {
  const int N = 1 << logN;
  const int lq = logN - 2;
  int lh = logN - 2;  // span of the first radix-4 stage: N/4
  __syncthreads();
  for (; lh >= 0; lh -= 2) {
    const int h = 1 << lh;
    for (int j = threadIdx.x; j < (G << lq); j += blockDim.x) {
      double2* xg = x + (j >> lq) * N;
      const int jj = j & ((1 << lq) - 1);
      const int pos = jj & (h - 1);
      const int i0 = ((jj - pos) << 2) + pos, i1 = i0 + h, i2 = i1 + h, i3 = i2 + h;
      const double2 w4 = twn(2 * (h - 1) + h + pos), w2 = twn(2 * (h - 1) + pos);
      const double2 x0 = xg[fsw(i0)], x1 = xg[fsw(i1)], x2 = xg[fsw(i2)], x3 = xg[fsw(i3)];
      const double2 t0 = cadd(x0, x2), t1 = cadd(x1, x3);
      double2 t2 = cmul(csub(x0, x2), w4);
      double2 t3 = cmul(csub(x1, x3), w4);
      t3 = make_double2(t3.y, -t3.x);  // * (-i)
      xg[fsw(i0)] = cadd(t0, t1);
      xg[fsw(i1)] = cmul(csub(t0, t1), w2);
      xg[fsw(i2)] = cadd(t2, t3);
      xg[fsw(i3)] = cmul(csub(t2, t3), w2);
    }
    __syncthreads();
  }
  if (lh == -1) {  // odd logN: final radix-2 stage, span 1, twiddle 1
    const int half = N >> 1;
    for (int j = threadIdx.x; j < G * half; j += blockDim.x) {
      double2* xg = x + (j >> (logN - 1)) * N;
      const int jj = j & (half - 1);
      const double2 a = xg[fsw(2 * jj)], b = xg[fsw(2 * jj + 1)];
      xg[fsw(2 * jj)] = cadd(a, b);
      xg[fsw(2 * jj + 1)] = csub(a, b);
    }
    __syncthreads();
  }
}

// inverse-sign DIT, input bit-reversed, output natural (unnormalised)
static __device__ void fft_dit_inv_multi(double2* x, int logN, int G, const StageTw twn) {
  const int N = 1 << logN;
  __syncthreads();
  int lh = 0;
  if (logN & 1) {
    const int half = N >> 1;
    for (int j = threadIdx.x; j < G * half; j += blockDim.x) {
      double2* xg = x + (j >> (logN - 1)) * N;
      const int jj = j & (half - 1);
      const double2 a = xg[fsw(2 * jj)], b = xg[fsw(2 * jj + 1)];
      xg[fsw(2 * jj)] = cadd(a, b);
      xg[fsw(2 * jj + 1)] = csub(a, b);
    }
    lh = 1;
    __syncthreads();
  }
  const int lq = logN - 2;
  for (; lh < logN; lh += 2) {
    const int h = 1 << lh;
    for (int j = threadIdx.x; j < (G << lq); j += blockDim.x) {
      double2* xg = x + (j >> lq) * N;
      const int jj = j & ((1 << lq) - 1);
      const int pos = jj & (h - 1);
      const int i0 = ((jj - pos) << 2) + pos, i1 = i0 + h, i2 = i1 + h, i3 = i2 + h;
      const double2 w1 = conj2(twn(2 * (h - 1) + pos)), w2 = conj2(twn(2 * (h - 1) + h + pos));
      const double2 a0 = xg[fsw(i0)], a1 = cmul(w1, xg[fsw(i1)]), a2 = xg[fsw(i2)], a3 = cmul(w1, xg[fsw(i3)]);
      const double2 b0 = cadd(a0, a1), b1 = csub(a0, a1), b2 = cadd(a2, a3), b3 = csub(a2, a3);
      const double2 c2 = cmul(w2, b2);
      double2 c3 = cmul(w2, b3);
      c3 = make_double2(-c3.y, c3.x);  // * (+i)
      xg[fsw(i0)] = cadd(b0, c2);
      xg[fsw(i2)] = csub(b0, c2);
      xg[fsw(i1)] = cadd(b1, c3);
      xg[fsw(i3)] = csub(b1, c3);
    }
    __syncthreads();
  }
}

// Per-stage twiddle table for fft_dif_fwd_multi / fft_dit_inv_multi: for the
// radix-4 stage of span h = 2^lh, W_2h^pos at sw[2(h-1) + pos] and W_4h^pos at
// sw[2(h-1) + h + pos] (pos < h), so a warp reads consecutive entries.  The
// entries do not depend on N (a transform of size N uses the first N - 2);
// built once per plan into global memory (OSPH_SW_GLOBAL entries).
