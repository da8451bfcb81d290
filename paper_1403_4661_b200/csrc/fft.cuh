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
