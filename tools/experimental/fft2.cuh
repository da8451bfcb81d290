// fft2.cuh -- register-blocked Bluestein convolution for power-of-two lengths
// N = N1 * N2 with N1, N2 <= 32 (N = 256, 512, 1024: every Bluestein ring up to
// L = 256 and most of L = 512).
//
// conv = IFFT(FFT(x) . bhat) in four register passes and three shared-memory
// exchanges (the radix-4 path in fft.cuh makes log4 N passes per transform):
//   S1  thread n2 < N2 : DFT_N1 over x[N2 n1 + n2], twiddle W_N^(n2 k1) -> Y[k1][n2]
//   S2  thread k1 < N1 : DFT_N2 over Y[k1][.] -> X[k1 + N1 k2] (natural order), times bhat
//   S3  same thread    : the inverse transform factored the other way round
//                        (m = N1 m1 + m2 with m2 = k1), so its first pass is a
//                        DFT_N2 over the registers S2 left -> twiddle W_N^-(m2 j1) -> Z[j1][m2]
//   S4  thread j1 < N2 : DFT_N1 over Z[j1][.] -> out[j1 + N2 j2], natural order
// Exchanges use a row pitch of (row length + 1) complex so the transposed
// reads are conflict-free.  Radix-2 DIF inside registers; all register indices
// are compile-time constants.
#pragma once
#include "../../paper_1403_4661_b200/csrc/common.cuh"

__constant__ double2 c_w32[32] = {
    {1, -0},
    {0.98078528040323043, -0.19509032201612825},
    {0.92387953251128674, -0.38268343236508978},
    {0.83146961230254524, -0.55557023301960218},
    {0.70710678118654757, -0.70710678118654746},
    {0.55557023301960229, -0.83146961230254524},
    {0.38268343236508984, -0.92387953251128674},
    {0.19509032201612833, -0.98078528040323043},
    {6.123233995736766e-17, -1},
    {-0.19509032201612819, -0.98078528040323043},
    {-0.38268343236508973, -0.92387953251128674},
    {-0.55557023301960196, -0.83146961230254546},
    {-0.70710678118654746, -0.70710678118654757},
    {-0.83146961230254535, -0.55557023301960218},
    {-0.92387953251128674, -0.38268343236508989},
    {-0.98078528040323043, -0.19509032201612861},
    {-1, -1.2246467991473532e-16},
    {-0.98078528040323043, 0.19509032201612836},
    {-0.92387953251128685, 0.38268343236508967},
    {-0.83146961230254546, 0.55557023301960196},
    {-0.70710678118654768, 0.70710678118654746},
    {-0.55557023301960218, 0.83146961230254524},
    {-0.38268343236509034, 0.92387953251128652},
    {-0.19509032201612866, 0.98078528040323032},
    {-1.8369701987210297e-16, 1},
    {0.1950903220161283, 0.98078528040323043},
    {0.38268343236509, 0.92387953251128663},
    {0.55557023301960184, 0.83146961230254546},
    {0.70710678118654735, 0.70710678118654768},
    {0.83146961230254524, 0.55557023301960218},
    {0.92387953251128652, 0.38268343236509039},
    {0.98078528040323032, 0.19509032201612872}
};

__host__ __device__ constexpr int bitrev_c(int v, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((v >> i) & 1) << (bits - 1 - i);
  return r;
}
__host__ __device__ constexpr int ilog2_c(int v) { return v <= 1 ? 0 : 1 + ilog2_c(v >> 1); }

// In-place radix-2 DIF DFT of R points (natural in, bit-reversed out); INV
// selects the + sign.  a[bitrev(k)] holds output k.
template <int R, bool INV>
__device__ __forceinline__ void dft_reg(double2 (&a)[R]) {
#pragma unroll
  for (int h = R / 2; h >= 1; h >>= 1) {
#pragma unroll
    for (int base = 0; base < R; base += 2 * h) {
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const double2 u = a[base + j], v = a[base + j + h];
        a[base + j] = cadd(u, v);
        const double2 d = csub(u, v);
        if (j == 0) {
          a[base + j + h] = d;
        } else {
          const double2 w = c_w32[j * (32 / (2 * h))];
          a[base + j + h] = INV ? cmul(d, conj2(w)) : cmul(d, w);
        }
      }
    }
  }
}

// W_N^e (forward sign) from the half-period table tw[j] = W_16384^j, j < 8192
// (N | 16384): W^(j + 8192) = -W^j
__device__ __forceinline__ double2 tw_n(const double2* __restrict__ tw, int N, int e) {
  const int j = (e & (N - 1)) * (16384 / N);
  const double2 w = __ldg(tw + (j & 8191));
  return j < 8192 ? w : make_double2(-w.x, -w.y);
}

// A length-R DFT computed by P = R/16 threads (P = 1 or 2, partner lane = lane ^ 1),
// each holding H = R/P points in registers.
//
// dft_split_dif: input natural halves (lower thread x[0..R/2), upper x[R/2..R)),
//   output: lower X[2k] at h[bitrev(k)], upper X[2k+1] at h[bitrev(k)] (P = 2);
//   P = 1: h[bitrev(k)] = X[k].
// dft_split_dit: input lower x[2k] at h[k], upper x[2k+1] at h[k] (P = 2; P = 1:
//   natural), output natural halves: lower X[j] at h[j], upper X[j + R/2] at h[j].
template <int R>
struct Split {
  static constexpr int P = R > 16 ? 2 : 1;
  static constexpr int H = R / P;
  static constexpr int LB = ilog2_c(H);
};

template <int R, bool INV>
__device__ __forceinline__ void dft_split_dif(double2 (&h)[Split<R>::H], bool upper) {
  if constexpr (Split<R>::P == 2) {
#pragma unroll
    for (int j = 0; j < R / 2; ++j) {
      const double2 mine = h[j];
      const double2 other = make_double2(__shfl_xor_sync(0xffffffffu, mine.x, 1), __shfl_xor_sync(0xffffffffu, mine.y, 1));
      if (!upper) {
        h[j] = cadd(mine, other);
      } else {
        const double2 d = csub(other, mine);
        const double2 w = c_w32[j * (32 / R)];
        h[j] = j == 0 ? d : (INV ? cmul(d, conj2(w)) : cmul(d, w));
      }
    }
  }
  dft_reg<Split<R>::H, INV>(h);
}

template <int R, bool INV>
__device__ __forceinline__ void dft_split_dit(double2 (&h)[Split<R>::H], bool upper) {
  constexpr int H = Split<R>::H, LB = Split<R>::LB;
  dft_reg<H, INV>(h);
#pragma unroll
  for (int k = 0; k < H; ++k)  // to natural order (static swaps)
    if (k < bitrev_c(k, LB)) {
      const double2 t = h[k];
      h[k] = h[bitrev_c(k, LB)];
      h[bitrev_c(k, LB)] = t;
    }
  if constexpr (Split<R>::P == 2) {
#pragma unroll
    for (int j = 0; j < H; ++j) {
      const double2 mine = h[j];
      const double2 other = make_double2(__shfl_xor_sync(0xffffffffu, mine.x, 1), __shfl_xor_sync(0xffffffffu, mine.y, 1));
      const double2 w = c_w32[j * (32 / R)];
      const double2 wj = INV ? conj2(w) : w;
      // lower: E + W O (E mine, O other); upper: E - W O (E other, O mine)
      h[j] = !upper ? cadd(mine, j == 0 ? other : cmul(other, wj)) : csub(other, j == 0 ? mine : cmul(mine, wj));
    }
  }
}

// Per-map buffer length (complex) for the exchanges of an N1 x N2 transform.// Per-map buffer length (complex) for the exchanges of an N1 x N2 transform.
template <int N1, int N2>
__host__ __device__ constexpr int conv2_stride() {
  return (N1 * (N2 + 1) > N2 * (N1 + 1) ? N1 * (N2 + 1) : N2 * (N1 + 1));
}

// Threads per map of bluestein_conv2 (32-point DFTs run on lane pairs).
template <int N1, int N2>
__host__ __device__ constexpr int conv2_tpm() {
  return N2 * Split<N1>::P > N1 * Split<N2>::P ? N2 * Split<N1>::P : N1 * Split<N2>::P;
}

// Bluestein circular convolution of one map held natural-order in xs[0..N)
// (xs has conv2_stride<N1,N2>() entries), kernel spectrum bh (natural order,
// includes 1/N).  Threads tm < conv2_tpm of the map take part (maps are
// aligned to whole pairs of lanes); every thread of the block must call it (it
// contains __syncthreads).  The result replaces xs[0..N) in natural order
// (visible to the whole block on return).
template <int N1, int N2>
__device__ __forceinline__ void bluestein_conv2(double2* xs, int tm, bool active, const double2* __restrict__ bh,
                                                const double2* __restrict__ tw) {
  constexpr int N = N1 * N2;
  constexpr int P1 = Split<N1>::P, H1 = Split<N1>::H, L1 = Split<N1>::LB;
  constexpr int P2 = Split<N2>::P, H2 = Split<N2>::H, L2 = Split<N2>::LB;
  // S1: column n2 = tm / P1 (half u1 = tm % P1 of the N1 rows)
  {
    const int n2 = tm / P1, u1 = tm % P1;
    const bool on = active && n2 < N2;
    double2 a[H1];
    if (on) {
#pragma unroll
      for (int i = 0; i < H1; ++i) a[i] = xs[N2 * (u1 * H1 + i) + n2];
    }
    __syncthreads();
    if (tm < N2 * P1) dft_split_dif<N1, false>(a, u1 == 1);  // whole pairs take part in the shuffles
    if (on) {
#pragma unroll
      for (int q = 0; q < H1; ++q) {
        const int k1 = P1 * q + u1;  // a[bitrev(q)] = Y[k1]
        const double2 v = a[bitrev_c(q, L1)];
        xs[k1 * (N2 + 1) + n2] = k1 == 0 ? v : cmul(v, tw_n(tw, N, n2 * k1));
      }
    }
  }
  __syncthreads();
  // S2 + bhat + S3: row k1 = m2 = tm / P2 (half u2 of the N2 columns)
  {
    const int k1 = tm / P2, u2 = tm % P2;
    const bool on = active && k1 < N1;
    double2 b[H2];
    if (on) {
#pragma unroll
      for (int i = 0; i < H2; ++i) b[i] = xs[k1 * (N2 + 1) + u2 * H2 + i];
    }
    __syncthreads();
    const bool part = tm < N1 * P2;
    if (part) dft_split_dif<N2, false>(b, u2 == 1);
    // X[k1 + N1 k2] with k2 = P2 q + u2 at b[bitrev(q)]: bring q to natural order and apply bhat
#pragma unroll
    for (int q = 0; q < H2; ++q)
      if (q < bitrev_c(q, L2)) {
        const double2 t = b[q];
        b[q] = b[bitrev_c(q, L2)];
        b[bitrev_c(q, L2)] = t;
      }
    if (on) {
#pragma unroll
      for (int q = 0; q < H2; ++q) b[q] = cmul(b[q], __ldg(bh + k1 + N1 * (P2 * q + u2)));
    }
    // inverse DFT over k2 (even / odd split across the pair): natural halves out
    if (part) dft_split_dit<N2, true>(b, u2 == 1);
    if (on) {
#pragma unroll
      for (int j = 0; j < H2; ++j) {
        const int j1 = u2 * H2 + j;
        const double2 v = b[j];
        xs[j1 * (N1 + 1) + k1] = j1 == 0 ? v : cmul(v, conj2(tw_n(tw, N, k1 * j1)));
      }
    }
  }
  __syncthreads();
  // S4: column j1 = tm / P1 (half of the N1 entries m2)
  {
    const int j1 = tm / P1, u1 = tm % P1;
    const bool on = active && j1 < N2;
    double2 d[H1];
    if (on) {
#pragma unroll
      for (int i = 0; i < H1; ++i) d[i] = xs[j1 * (N1 + 1) + u1 * H1 + i];
    }
    if (tm < N2 * P1) dft_split_dif<N1, true>(d, u1 == 1);
    __syncthreads();  // every Z read above is done
    if (on) {
#pragma unroll
      for (int q = 0; q < H1; ++q) xs[j1 + N2 * (P1 * q + u1)] = d[bitrev_c(q, L1)];
    }
  }
  __syncthreads();
}
