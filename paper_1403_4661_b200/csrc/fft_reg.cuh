// fft_reg.cuh -- register-resident Bluestein convolution for the ring DFTs.
//
// The shared-memory radix-4 transform of fft.cuh moves every element through
// shared memory once per stage (10 stage passes per 1024-point convolution)
// and is bound by shared-memory bandwidth, not by the fp64 pipe
// (profiles/ringinv_r02_full.txt: fp64 pipe 26% busy).  Here a length
// N = N1 * N2 transform is two passes of register-resident radix-N1 / radix-N2
// butterflies (N1, N2 in {16, 32}; twiddles of the butterflies are immediates),
// one small group of T = N2 threads per transform, and the whole circular
// convolution
//   y = IFFT_N( FFT_N(x) * H )
// needs only TWO exchanges through shared memory:
//   pass 1   thread n2: radix-N1 DIF over n1 of x[n1 N2 + n2]  -> k1 (bit-reversed registers)
//            times W_N^(n2 k1), written to Y[k1][n2]
//   pass 2   task k1: radix-N2 DIF over n2 -> X[k1 + N1 k2] (k2 bit-reversed registers),
//            times H (natural order in global memory, coalesced over k1),
//            radix-N2 inverse DIT over k2 (bit-reversed in, natural out),
//            times conj W_N^(n2 k1), back to Y[k1][n2]
//   pass 1'  thread n2: radix-N1 inverse DIT over k1 -> y[n1 N2 + n2]
// The exchanges are local to the group (a warp or half a warp): __syncwarp only.
// Y rows are padded to N2 + 1 entries, which makes both access directions
// bank-conflict free for 16-byte elements.
//
// Bluestein inputs are zero beyond n <= N/2, so the first DIF stage of pass 1
// and the last DIT stage of pass 1' are pruned (ZERO_UPPER / LOWER_ONLY).
#pragma once
#include "common.cuh"

__host__ __device__ constexpr int rf_brev(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}
__host__ __device__ constexpr int rf_log2(int v) { return v <= 1 ? 0 : 1 + rf_log2(v >> 1); }

// v * e^{-+ 2 pi i j / 32}, 0 <= j < 16 (j is a compile-time constant after unrolling)
template <bool INV>
__device__ __forceinline__ double2 rf_mul_w32(double2 v, int j) {
  constexpr double h = 0.70710678118654752440;
  if (j == 0) return v;
  if (j == 8) return INV ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
  if (j == 4) return INV ? make_double2((v.x - v.y) * h, (v.x + v.y) * h) : make_double2((v.x + v.y) * h, (v.y - v.x) * h);
  if (j == 12)
    return INV ? make_double2(-(v.x + v.y) * h, (v.x - v.y) * h) : make_double2((v.y - v.x) * h, -(v.x + v.y) * h);
  double c = 1.0, s = 0.0;  // cos, sin of 2 pi j / 32
  switch (j) {
    case 1: c = 0.98078528040323044913; s = 0.19509032201612826785; break;
    case 2: c = 0.92387953251128675613; s = 0.38268343236508977173; break;
    case 3: c = 0.83146961230254523708; s = 0.55557023301960222474; break;
    case 5: c = 0.55557023301960222474; s = 0.83146961230254523708; break;
    case 6: c = 0.38268343236508977173; s = 0.92387953251128675613; break;
    case 7: c = 0.19509032201612826785; s = 0.98078528040323044913; break;
    case 9: c = -0.19509032201612826785; s = 0.98078528040323044913; break;
    case 10: c = -0.38268343236508977173; s = 0.92387953251128675613; break;
    case 11: c = -0.55557023301960222474; s = 0.83146961230254523708; break;
    case 13: c = -0.83146961230254523708; s = 0.55557023301960222474; break;
    case 14: c = -0.92387953251128675613; s = 0.38268343236508977173; break;
    case 15: c = -0.98078528040323044913; s = 0.19509032201612826785; break;
    default: break;
  }
  return INV ? make_double2(fma(v.x, c, -v.y * s), fma(v.y, c, v.x * s))
             : make_double2(fma(v.x, c, v.y * s), fma(v.y, c, -v.x * s));
}

// One radix-2 stage of half-size S = 2^LS on R registers (every index is a compile-time constant).
// MODE 0: a' = a + c, c' = (a - c) w (DIF); MODE 1: c = 0 known, c' = a w (pruned DIF);
// MODE 2: c w first, a' = a + cw, c' = a - cw (DIT); MODE 3: DIT, a' only.
template <int R, int LS, bool INV, int MODE>
__device__ __forceinline__ void rf_stage(double2 (&v)[R]) {
  constexpr int S = 1 << LS;
#pragma unroll
  for (int i = 0; i < R / 2; ++i) {
    const int b = (i / S) * 2 * S, j = i % S;
    if (MODE == 0) {
      const double2 a = v[b + j], c = v[b + j + S];
      v[b + j] = cadd(a, c);
      v[b + j + S] = rf_mul_w32<INV>(csub(a, c), j * (16 / S));
    } else if (MODE == 1) {
      v[b + j + S] = rf_mul_w32<INV>(v[b + j], j * (16 / S));
    } else {
      const double2 a = v[b + j], c = rf_mul_w32<INV>(v[b + j + S], j * (16 / S));
      v[b + j] = cadd(a, c);
      if (MODE == 2) v[b + j + S] = csub(a, c);
    }
  }
}

// Decimation in frequency, natural order in, v[i] = X[brev(i)] out.
// ZERO_UPPER: v[R/2..R) are known zeros on entry (their values are ignored).
template <int R, bool INV, bool ZERO_UPPER, int LS = rf_log2(R) - 1>
__device__ __forceinline__ void rf_dif(double2 (&v)[R]) {
  rf_stage<R, LS, INV, (ZERO_UPPER && LS == rf_log2(R) - 1) ? 1 : 0>(v);
  if constexpr (LS > 0) rf_dif<R, INV, ZERO_UPPER, LS - 1>(v);
}

// Decimation in time, v[i] = X[brev(i)] in, natural order out.
// LOWER_ONLY: only v[0..R/2) are needed on exit (the rest is left undefined).
template <int R, bool INV, bool LOWER_ONLY, int LS = 0>
__device__ __forceinline__ void rf_dit(double2 (&v)[R]) {
  rf_stage<R, LS, INV, (LOWER_ONLY && LS == rf_log2(R) - 1) ? 3 : 2>(v);
  if constexpr (LS < rf_log2(R) - 1) rf_dit<R, INV, LOWER_ONLY, LS + 1>(v);
}

// One circular convolution of length N = N1 * N2 by a group of T = N2 threads.
template <int N1, int N2>
struct RegConv {
  static constexpr int N = N1 * N2;
  static constexpr int T = N2;        // threads per transform
  static constexpr int Q = N1 / N2;   // pass-2 tasks per thread
  static constexpr int LD = N2 + 1;   // padded row length of the exchange matrix Y[N1][LD]
  static constexpr int RS = N1 * LD;  // double2 entries of Y (and of the twiddle table)
  static_assert(N1 >= N2 && N1 % N2 == 0 && N1 <= 32 && N2 >= 8, "unsupported factorisation");

  // v[n1] = x[n1 N2 + tid] for n1 < N1/2 on entry (x is zero beyond N/2);
  // v[n1] = y[n1 N2 + tid] for n1 < N1/2 on exit.  Y: this group's exchange
  // matrix; TW[k1 LD + n2] = e^{-2 pi i k1 n2 / N}; H[k]: kernel spectrum,
  // natural order (any 1/N factor folded in), in shared memory like TW.  All
  // lanes of the warp call it.
  // FULL: the input fills all N1 registers and every output is produced (the
  // two half-size convolutions of a 2N-point Bluestein ring, ringdft.cu).
  template <bool FULL = false>
  __device__ static __forceinline__ void run(double2 (&v)[N1], double2* Y, const double2* TW, const double2* H,
                                            int tid) {
    constexpr int L1 = rf_log2(N1), L2 = rf_log2(N2);
    rf_dif<N1, false, !FULL>(v);
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      const int k1 = rf_brev(i, L1);
      Y[k1 * LD + tid] = cmul(v[i], TW[k1 * LD + tid]);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int k1 = tid + q * T;
      double2 u[N2];
#pragma unroll
      for (int n2 = 0; n2 < N2; ++n2) u[n2] = Y[k1 * LD + n2];
      rf_dif<N2, false, false>(u);
#pragma unroll
      for (int i = 0; i < N2; ++i) u[i] = cmul(u[i], H[k1 + N1 * rf_brev(i, L2)]);
      rf_dit<N2, true, false>(u);
#pragma unroll
      for (int n2 = 0; n2 < N2; ++n2) Y[k1 * LD + n2] = cmul(u[n2], conj2(TW[k1 * LD + n2]));
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < N1; ++i) v[i] = Y[rf_brev(i, L1) * LD + tid];
    rf_dit<N1, true, !FULL>(v);
  }
};
