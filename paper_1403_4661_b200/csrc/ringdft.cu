// ringdft.cu -- per-ring odd-length DFTs (lengths n = 2k+1).
//
// Inverse (synthesis) side: fold the 2L-1 tones G_(+-m)(theta_k) of every ring
// into its n native bins and apply an inverse DFT -- the reference's
// _fold_bins + per-ring (n/2pi) * ifft (transform.py:204-218, 334-344).  The
// 2pi of G and the 1/2pi of the synthesis cancel, so G is consumed raw.
//
// Forward (analysis) side: one forward DFT per ring (transform.py:439, the
// "spectral" method), scattered straight into the order-major RHS layout the
// peeling sweep consumes: R[pos(m, k-m)][+/-][b] = (2pi/n) X_k[+-m mod n]
// (transform.py:445-449).
//
// n <= OSPH_DIRECT_MAX: direct O(n^2) DFT from a roots table.  Longer rings:
// Bluestein (chirp-z) with a power-of-two FFT in shared memory.  A block
// handles one ring and a run of maps, transforming several maps per pass so
// the FFT stage barriers are shared; global accesses run map-fastest, which
// is the contiguous direction of G and R.
#include <cooperative_groups.h>
#include <cstdlib>

#include "fft.cuh"
#include "fft_reg.cuh"
#include "plan.cuh"

namespace cg = cooperative_groups;

#define RING_THREADS 256
#define RING_SMEM_BUDGET (48 * 1024)  // measured (config 2): 48 KB + 16 waves beats 96 KB + 4 waves by 11-15%

// Fold G (layout [m][k][4B]) of ring k, map b into bin t (t < n).
__device__ __forceinline__ double2 fold_bin(const double* __restrict__ G, int L, int B, int k, int n, int b, int t) {
  const int64_t mstride = (int64_t)L * 4 * B;
  const double* gk = G + ((int64_t)k * 4 * B + 4 * b);
  double re = 0.0, im = 0.0;
  for (int m = t; m < L; m += n) {  // +m tones: bin m mod n
    const double2 v = __ldg(reinterpret_cast<const double2*>(gk + m * mstride));
    re += v.x;
    im += v.y;
  }
  for (int m = (t == 0 ? n : n - t); m < L; m += n) {  // -m tones, m >= 1: bin -m mod n
    const double2 v = __ldg(reinterpret_cast<const double2*>(gk + m * mstride + 2));
    if (m & 1) {
      re -= v.x;
      im -= v.y;
    } else {
      re += v.x;
      im += v.y;
    }
  }
  return make_double2(re, im);
}

// Bluestein circular convolution of Gr sequences (natural order, swizzled):
// DIF forward FFT -> times the kernel spectrum (stored bit-reversed, /N) ->
// DIT inverse FFT; natural order out, no bit-reversal passes.
__device__ __forceinline__ void bluestein_convolve(double2* xs, int logN, int Gr, const StageTw twn,
                                                   const double2* __restrict__ bh_br) {
  fft_dif_fwd_multi(xs, logN, Gr, twn);
  const int N = 1 << logN;
  for (int idx = threadIdx.x; idx < (Gr << logN); idx += blockDim.x) {
    const int q = idx & (N - 1);
    double2* e = xs + (idx - q) + fsw(q);
    *e = cmul(*e, __ldg(bh_br + q));
  }
  fft_dit_inv_multi(xs, logN, Gr, twn);
}

// For Gr maps: x *= bhat (natural order), then bit-reverse every map in place.
__device__ __forceinline__ void mul_and_bitrev_multi(double2* x, const double2* __restrict__ bh, int N, int logN,
                                                     int Gr) {
  for (int idx = threadIdx.x; idx < (Gr << logN); idx += blockDim.x) x[idx] = cmul(x[idx], __ldg(bh + (idx & (N - 1))));
  __syncthreads();
  for (int idx = threadIdx.x; idx < (Gr << logN); idx += blockDim.x) {
    const int q = idx & (N - 1);
    const int r = bitrev(q, logN);
    if (q < r) {
      double2* xg = x + (idx - q);
      const double2 a = xg[q];
      xg[q] = xg[r];
      xg[r] = a;
    }
  }
}

__global__ void __launch_bounds__(RING_THREADS) k_ring_inverse_bluestein(
    int L, int B, int maps_per_block, const int* __restrict__ rings, const int* __restrict__ fft_n,
    const int64_t* __restrict__ chirp_off, const int64_t* __restrict__ bhat_off, const double2* __restrict__ chirp_all,
    const double2* __restrict__ bhat_all, const double2* __restrict__ gsw, const double* __restrict__ G,
    double2* __restrict__ samples, int smem_cplx) {
  extern __shared__ double2 sm[];
  const int k = rings[blockIdx.x];
  const int n = 2 * k + 1;
  const int N = fft_n[k];
  const int logN = 31 - __clz(N);
  // Gr transforms of length N after the short-span twiddles: a size-N transform
  // reads stage-table entries < N only, so the data start right after them
  const int tw_cnt = min(N, OSPH_SW_SMEM);
  double2* xs = sm + tw_cnt;
  load_stage_twiddles_smem(sm, logN, gsw);
  const StageTw twn{sm, gsw};
  const double2* chirp = chirp_all + chirp_off[k];
  const double2* bh = bhat_all + bhat_off[k] + N;  // inverse-direction kernel
  const int b_first = blockIdx.y * maps_per_block;
  const int b_last = min(B, b_first + maps_per_block);
  const int Gmax = max(1, (smem_cplx - tw_cnt) >> logN);
  for (int b0 = b_first; b0 < b_last; b0 += Gmax) {
    const int Gr = min(Gmax, b_last - b0);
    for (int idx = threadIdx.x; idx < Gr * N; idx += blockDim.x) {  // map-fastest reads of G
      const int g = idx % Gr, t = idx / Gr;
      double2 v = make_double2(0.0, 0.0);
      if (t < n) v = cmul(fold_bin(G, L, B, k, n, b0 + g, t), __ldg(chirp + t));
      xs[(g << logN) + fsw(t)] = v;
    }
    bluestein_convolve(xs, logN, Gr, twn, bh);
    for (int idx = threadIdx.x; idx < Gr * n; idx += blockDim.x) {  // contiguous ring writes per map
      const int g = idx / n, j = idx - g * n;
      samples[(int64_t)(b0 + g) * L * L + (int64_t)k * k + j] = cmul(xs[(g << logN) + fsw(j)], __ldg(chirp + j));
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(RING_THREADS) k_ring_inverse_direct(int L, int B, int maps_per_block, int k0,
                                                                      const double2* __restrict__ roots,
                                                                      const double* __restrict__ G,
                                                                      double2* __restrict__ samples) {
  __shared__ double2 bins[16][OSPH_DIRECT_MAX + 1];
  __shared__ double2 part[RING_THREADS];  // per-part fold sums (deterministic order)
  const int k = k0 + blockIdx.x;
  const int n = 2 * k + 1;
  const int b_first = blockIdx.y * maps_per_block;
  const int b_last = min(B, b_first + maps_per_block);
  const double2* rt = roots + (int64_t)k * k;
  for (int b0 = b_first; b0 < b_last; b0 += 16) {
    const int Gr = min(16, b_last - b0);
    // fold: short rings gather up to 2L tones per bin.  Deterministic: bin (g, t)
    // is split into P interleaved parts (i = p, p + P, ... of its +m and -m tone
    // lists), one thread sums a part in order, and the parts are added in p order
    // (no floating-point atomics: bitwise reproducible like the reference).
    const int items = Gr * n;
    const int P = max(1, RING_THREADS / items);
    const int64_t mstride = (int64_t)L * 4 * B;
    for (int idx = threadIdx.x; idx < items * P; idx += blockDim.x) {
      const int p = idx / items, item = idx - p * items;
      const int t = item / Gr, g = item - t * Gr;  // map fastest: neighbouring threads read neighbouring maps
      const double* gk = G + ((int64_t)k * 4 * B + 4 * (b0 + g));
      double re = 0.0, im = 0.0;
      for (int m = t + p * n; m < L; m += P * n) {  // +m tones: bin m mod n
        const double2 v = __ldg(reinterpret_cast<const double2*>(gk + m * mstride));
        re += v.x;
        im += v.y;
      }
      for (int m = (t == 0 ? n : n - t) + p * n; m < L; m += P * n) {  // -m tones (m >= 1): bin -m mod n
        const double2 v = __ldg(reinterpret_cast<const double2*>(gk + m * mstride + 2));
        if (m & 1) {
          re -= v.x;
          im -= v.y;
        } else {
          re += v.x;
          im += v.y;
        }
      }
      if (P == 1) bins[g][t] = make_double2(re, im);
      else part[idx] = make_double2(re, im);
    }
    __syncthreads();
    if (P > 1) {
      for (int item = threadIdx.x; item < items; item += blockDim.x) {
        const int t = item / Gr, g = item - t * Gr;
        double2 acc = part[item];
        for (int p = 1; p < P; ++p) acc = cadd(acc, part[p * items + item]);
        bins[g][t] = acc;
      }
      __syncthreads();
    }
    for (int idx = threadIdx.x; idx < Gr * n; idx += blockDim.x) {
      const int g = idx / n, j = idx - g * n;
      double re = 0.0, im = 0.0;
      int r = 0;
      for (int t = 0; t < n; ++t) {  // e^{+2 pi i t j / n}
        const double2 w = rt[r];
        const double2 v = bins[g][t];
        re += v.x * w.x - v.y * w.y;
        im += v.x * w.y + v.y * w.x;
        r += j;
        if (r >= n) r -= n;
      }
      samples[(int64_t)(b0 + g) * L * L + (int64_t)k * k + j] = make_double2(re, im);
    }
    __syncthreads();
  }
}

// Scatter Gr ring spectra (forward sign, unnormalised; X[g][q] at x[(g<<lstride) + q])
// into the RHS layout, map-fastest.
template <bool SWZ>
__device__ __forceinline__ void scatter_rhs_multi(const double2* X, int lstride, int L, int lgG, int k, int n, int b0,
                                                  int Gr, double2* __restrict__ R) {
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  const double scale = OSPH_TWO_PI / (double)n;
  for (int idx = threadIdx.x; idx < Gr * (k + 1); idx += blockDim.x) {
    const int g = idx % Gr, m = idx / Gr;
    const int qn = m == 0 ? 0 : n - m;
    const double2 xp = X[(g << lstride) + (SWZ ? fsw(m) : m)];
    const double2 xn = X[(g << lstride) + (SWZ ? fsw(qn) : qn)];
    const int64_t base = r_index(packed_pos(L, m, k - m), 0, b0 + g, lgG, npos);
    R[base] = make_double2(scale * xp.x, scale * xp.y);
    // order 0 solves its + column only (f_{l,-0} = f_{l,0}, transform.py:451): its - slot
    // starts at zero and collects the sweep's -tone corrections that alias to bin 0
    // (s = 0 mod 2k+1), folded into the + slot before order 0 is solved (sweep.cu)
    R[base + (1 << lgG)] = m == 0 ? make_double2(0.0, 0.0) : make_double2(scale * xn.x, scale * xn.y);
  }
}

__global__ void __launch_bounds__(RING_THREADS) k_ring_forward_bluestein(
    int L, int B, int maps_per_block, const int* __restrict__ rings, const int* __restrict__ fft_n,
    const int64_t* __restrict__ chirp_off, const int64_t* __restrict__ bhat_off, const double2* __restrict__ chirp_all,
    const double2* __restrict__ bhat_all, const double2* __restrict__ gsw, const double2* __restrict__ samples,
    double2* __restrict__ R, int smem_cplx, int bofs, int bend, int lgG) {
  extern __shared__ double2 sm[];
  const int k = rings[blockIdx.x];
  const int n = 2 * k + 1;
  const int N = fft_n[k];
  const int logN = 31 - __clz(N);
  // Gr transforms of length N after the short-span twiddles: a size-N transform
  // reads stage-table entries < N only, so the data start right after them
  const int tw_cnt = min(N, OSPH_SW_SMEM);
  double2* xs = sm + tw_cnt;
  load_stage_twiddles_smem(sm, logN, gsw);
  const StageTw twn{sm, gsw};
  const double2* chirp = chirp_all + chirp_off[k];
  const double2* bh = bhat_all + bhat_off[k];  // forward-direction kernel
  // maps [bofs, bend) of a batch of B (R keeps the batch stride B)
  const int b_first = bofs + blockIdx.y * maps_per_block;
  const int b_last = min(bend, b_first + maps_per_block);
  const int Gmax = max(1, (smem_cplx - tw_cnt) >> logN);
  for (int b0 = b_first; b0 < b_last; b0 += Gmax) {
    const int Gr = min(Gmax, b_last - b0);
    for (int idx = threadIdx.x; idx < (Gr << logN); idx += blockDim.x) {  // contiguous ring reads per map
      const int g = idx >> logN, t = idx & (N - 1);
      double2 v = make_double2(0.0, 0.0);
      if (t < n) v = cmul(__ldg(samples + (int64_t)(b0 + g) * L * L + (int64_t)k * k + t), conj2(__ldg(chirp + t)));
      xs[(g << logN) + fsw(t)] = v;
    }
    bluestein_convolve(xs, logN, Gr, twn, bh);
    for (int idx = threadIdx.x; idx < (Gr << logN); idx += blockDim.x) {
      const int t = idx & (N - 1);
      if (t < n) xs[(idx - t) + fsw(t)] = cmul(xs[(idx - t) + fsw(t)], conj2(__ldg(chirp + t)));
    }
    __syncthreads();
    scatter_rhs_multi<true>(xs, logN, L, lgG, k, n, b0, Gr, R);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(RING_THREADS) k_ring_forward_direct(int L, int B, int maps_per_block,
                                                                      const double2* __restrict__ roots,
                                                                      const double2* __restrict__ samples,
                                                                      double2* __restrict__ R, int bofs, int bend,
                                                                      int lgG) {
  __shared__ double2 xin[16][OSPH_DIRECT_MAX + 1];
  __shared__ double2 X[16][64];
  const int k = blockIdx.x;
  const int n = 2 * k + 1;
  const int b_first = bofs + blockIdx.y * maps_per_block;
  const int b_last = min(bend, b_first + maps_per_block);
  const double2* rt = roots + (int64_t)k * k;
  for (int b0 = b_first; b0 < b_last; b0 += 16) {
    const int Gr = min(16, b_last - b0);
    for (int idx = threadIdx.x; idx < Gr * n; idx += blockDim.x) {
      const int g = idx / n, t = idx - g * n;
      xin[g][t] = samples[(int64_t)(b0 + g) * L * L + (int64_t)k * k + t];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < Gr * n; idx += blockDim.x) {
      const int g = idx / n, q = idx - g * n;
      double re = 0.0, im = 0.0;
      int r = 0;
      for (int t = 0; t < n; ++t) {  // e^{-2 pi i q t / n}
        const double2 w = rt[r];
        const double2 v = xin[g][t];
        re += v.x * w.x + v.y * w.y;
        im += v.y * w.x - v.x * w.y;
        r += q;
        if (r >= n) r -= n;
      }
      X[g][q] = make_double2(re, im);
    }
    __syncthreads();
    scatter_rhs_multi<false>(&X[0][0], 6, L, lgG, k, n, b0, Gr, R);
    __syncthreads();
  }
}


static int maps_per_block_for(int B, int rings);

// ---------------------------------------------------------------------------
// Register-resident Bluestein rings (fft_reg.cuh): FFT sizes 256, 512, 1024.
// A block is REG_WARPS warps; a group of T = N2 threads (a warp, or half a
// warp) convolves one map's ring, so a block iteration covers
// REG_WARPS * 32 / T maps.  Global accesses that are contiguous per map
// (samples) go straight between registers and global memory, coalesced over
// the group's lanes; the map-fastest arrays (G, R) are staged through the
// group's exchange matrix by the whole block.
// one 32-byte read-only load (sm_100: ld.global.nc.v4.f64); p is 32-byte aligned
__device__ __forceinline__ double4 ldg_f64x4(const double* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];\n" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

#define REG_WARPS 4
#define REG_THREADS (REG_WARPS * 32)

__device__ __forceinline__ int reg_rtw_offset(int N) { return N == 256 ? 0 : (N == 512 ? 272 : 816); }

// Shared memory of a block: [TW: RS][H: N][chirp: N/2][one exchange matrix of RS entries per group].
template <int N1, int N2>
__device__ __forceinline__ double2* reg_stage_tables(double2* sm, int n, const double2* __restrict__ chirp,
                                                     const double2* __restrict__ bh, const double2* __restrict__ rtw) {
  using C = RegConv<N1, N2>;
  for (int i = threadIdx.x; i < C::RS; i += blockDim.x) sm[i] = __ldg(rtw + reg_rtw_offset(C::N) + i);
  for (int i = threadIdx.x; i < C::N; i += blockDim.x) sm[C::RS + i] = __ldg(bh + i);
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[C::RS + C::N + i] = __ldg(chirp + i);
  return sm + C::RS + C::N + C::N / 2;
}

template <int N1, int N2>
__device__ __forceinline__ void ring_inverse_reg(int L, int B, int k, int b_first, int b_last, double2* sm,
                                                 const double2* __restrict__ chirp, const double2* __restrict__ bh,
                                                 const double2* __restrict__ rtw, const double* __restrict__ G,
                                                 double2* __restrict__ samples) {
  using C = RegConv<N1, N2>;
  constexpr int GPW = 32 / C::T;  // groups (maps) per warp
  const int n = 2 * k + 1;
  const int nwarps = blockDim.x >> 5;
  const int gmax = nwarps * GPW;
  const double2* tw = sm;
  const double2* hs = sm + C::RS;
  const double2* cs = sm + C::RS + C::N;
  double2* ys = reg_stage_tables<N1, N2>(sm, n, chirp, bh, rtw);
  const int lane = threadIdx.x & 31, g = (threadIdx.x >> 5) * GPW + lane / C::T, tid = lane % C::T;
  double2* Y = ys + C::RS * g;
  // Fold.  The tones m = t (mod n) feed bin t with their + half and bin -t with their
  // - half, so one thread per (residue t, map) reads both halves as ONE 32-byte load per
  // tone and keeps two sums: P[t] (+ halves) and M[t] (- halves, sign (-1)^m, m >= 1),
  // in increasing m (fixed order: bitwise reproducible).  Bin t = P[t] + M[-t mod n].
  // P sits at Y[0..n), M at Y[n..2n) of the map's exchange matrix (2n <= N <= RS).
  const int nres = min(n, L);  // residues that hold a tone
  const int64_t mstride = (int64_t)L * 4 * B;
  for (int b0 = b_first; b0 < b_last; b0 += gmax) {
    const int Gr = min(gmax, b_last - b0);
    const int items = Gr * nres;
    const double* gbase = G + ((int64_t)k * 4 * B + 4 * b0);
    if (n >= L) {  // one tone per residue: four independent loads in flight per thread
      for (int i0 = threadIdx.x; i0 < items; i0 += 4 * blockDim.x) {
        double4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int idx = i0 + u * blockDim.x;
          if (idx < items) {
            const int gg = idx % Gr, t = idx / Gr;
            q[u] = ldg_f64x4(gbase + 4 * gg + t * mstride);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int idx = i0 + u * blockDim.x;
          if (idx < items) {
            const int gg = idx % Gr, t = idx / Gr;
            double2* Yg = ys + C::RS * gg;
            Yg[t] = make_double2(q[u].x, q[u].y);
            Yg[n + t] = t == 0 ? make_double2(0.0, 0.0)
                               : ((t & 1) ? make_double2(-q[u].z, -q[u].w) : make_double2(q[u].z, q[u].w));
          }
        }
      }
    } else {
      for (int idx = threadIdx.x; idx < items; idx += blockDim.x) {
        const int gg = idx % Gr, t = idx / Gr;
        const double* gk = gbase + 4 * gg;
        double pr = 0.0, pi = 0.0, mr = 0.0, mi = 0.0;
        for (int m = t; m < L; m += n) {
          const double4 q = ldg_f64x4(gk + m * mstride);
          pr += q.x;
          pi += q.y;
          if (m > 0) {
            if (m & 1) {
              mr -= q.z;
              mi -= q.w;
            } else {
              mr += q.z;
              mi += q.w;
            }
          }
        }
        double2* Yg = ys + C::RS * gg;
        Yg[t] = make_double2(pr, pi);
        Yg[n + t] = make_double2(mr, mi);
      }
    }
    __syncthreads();
    double2 v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1 / 2; ++n1) {
      const int t = n1 * N2 + tid;
      v[n1] = make_double2(0.0, 0.0);
      if (t < n && g < Gr) {
        const int r = t == 0 ? 0 : n - t;
        const double2 a = t < nres ? Y[t] : make_double2(0.0, 0.0);
        const double2 b = r < nres ? Y[n + r] : make_double2(0.0, 0.0);
        v[n1] = cmul(cadd(a, b), cs[t]);
      }
    }
    __syncwarp();
    C::run(v, Y, tw, hs, tid);
    if (g < Gr) {
      double2* out = samples + (int64_t)(b0 + g) * L * L + (int64_t)k * k;
#pragma unroll
      for (int n1 = 0; n1 < N1 / 2; ++n1) {
        const int t = n1 * N2 + tid;
        if (t < n) out[t] = cmul(v[n1], cs[t]);
      }
    }
    __syncthreads();  // the next iteration's fold overwrites the exchange matrices
  }
}

// FFT size 2048 (rings 513 <= n <= 1023): the input is zero beyond n < 1024, so the first
// DIF stage splits the 2048-point transform into two 1024-point ones without any
// arithmetic on the upper half -- even bins: FFT_1024(a), odd bins: FFT_1024(a W_2048^t) --
// and the last DIT stage needs y_t = E_t + conj(W_2048^t) O_t for t < n only.  A PAIR of
// warps owns one map's ring: warp 0 convolves a with the even half of the kernel spectrum,
// warp 1 convolves a W^t with the odd half, applies conj(W^t) and hands its half over
// through its exchange matrix.  Shared memory: [TW: RS][chirp: 1024][one matrix per warp];
// the kernel spectrum halves (16 KB each, shared by every map) are read through L1.
// tw16k[j] = e^{-2 pi i j / 16384}, so W_2048^t = tw16k[8 t].
__device__ __forceinline__ void reg_pair_sync(int pair) {  // REG_WARPS = 4: two pairs, barriers 1 and 2
  if (pair == 0) asm volatile("bar.sync 1, 64;\n" ::: "memory");
  else asm volatile("bar.sync 2, 64;\n" ::: "memory");
}

__device__ __forceinline__ void ring_inverse_reg2(int L, int B, int k, int b_first, int b_last, double2* sm,
                                                  const double2* __restrict__ chirp, const double2* __restrict__ bh,
                                                  const double2* __restrict__ rtw, const double2* __restrict__ tw16k,
                                                  const double* __restrict__ G, double2* __restrict__ samples) {
  using C = RegConv<32, 32>;
  const int n = 2 * k + 1;
  const int nwarps = blockDim.x >> 5, gmax = nwarps >> 1;  // maps per block iteration
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, pair = warp >> 1, half = warp & 1;
  double2* tw = sm;
  double2* cs = sm + C::RS;
  double2* ys = sm + C::RS + 1024;
  for (int i = threadIdx.x; i < C::RS; i += blockDim.x) tw[i] = __ldg(rtw + reg_rtw_offset(1024) + i);
  for (int i = threadIdx.x; i < n; i += blockDim.x) cs[i] = __ldg(chirp + i);
  double2* YA = ys + C::RS * (2 * pair);      // P sums (fold), then warp 0's exchange matrix
  double2* YB = ys + C::RS * (2 * pair + 1);  // M sums (fold), then warp 1's exchange matrix
  double2* Y = half ? YB : YA;
  const double2* H = bh + half * 1024;  // even / odd bins of the inverse-direction kernel spectrum
  const int nres = min(n, L);
  const int64_t mstride = (int64_t)L * 4 * B;
  for (int b0 = b_first; b0 < b_last; b0 += gmax) {
    const int Gr = min(gmax, b_last - b0);
    const double* gbase = G + ((int64_t)k * 4 * B + 4 * b0);
    for (int idx = threadIdx.x; idx < Gr * nres; idx += blockDim.x) {  // fold as ring_inverse_reg: P and M sums
      const int gg = idx % Gr, t = idx / Gr;
      double pr = 0.0, pi = 0.0, mr = 0.0, mi = 0.0;
      for (int m = t; m < L; m += n) {
        const double4 q = ldg_f64x4(gbase + 4 * gg + m * mstride);
        pr += q.x;
        pi += q.y;
        if (m > 0) {
          mr += (m & 1) ? -q.z : q.z;
          mi += (m & 1) ? -q.w : q.w;
        }
      }
      ys[C::RS * (2 * gg) + t] = make_double2(pr, pi);
      ys[C::RS * (2 * gg + 1) + t] = make_double2(mr, mi);
    }
    __syncthreads();
    double2 v[32];
#pragma unroll
    for (int n1 = 0; n1 < 32; ++n1) {
      const int t = n1 * 32 + lane;
      v[n1] = make_double2(0.0, 0.0);
      if (t < n && pair < Gr) {
        const int r = t == 0 ? 0 : n - t;
        const double2 a = t < nres ? YA[t] : make_double2(0.0, 0.0);
        const double2 b = r < nres ? YB[r] : make_double2(0.0, 0.0);
        v[n1] = cmul(cadd(a, b), cs[t]);
        if (half) v[n1] = cmul(v[n1], __ldg(tw16k + 8 * t));
      }
    }
    reg_pair_sync(pair);  // both warps have read the fold sums
    C::run<true>(v, Y, tw, H, lane);
    __syncwarp();
    if (half) {
#pragma unroll
      for (int n1 = 0; n1 < 32; ++n1) {
        const int t = n1 * 32 + lane;
        if (t < n) YB[t] = cmul(v[n1], conj2(__ldg(tw16k + 8 * t)));
      }
    }
    reg_pair_sync(pair);
    if (!half && pair < Gr) {
      double2* out = samples + (int64_t)(b0 + pair) * L * L + (int64_t)k * k;
#pragma unroll
      for (int n1 = 0; n1 < 32; ++n1) {
        const int t = n1 * 32 + lane;
        if (t < n) out[t] = cmul(cadd(v[n1], YB[t]), cs[t]);
      }
    }
    __syncthreads();  // the next iteration's fold overwrites the exchange matrices
  }
}

__device__ __forceinline__ void ring_forward_reg2(int L, int k, int b_first, int b_last, int lgG, double2* sm,
                                                  const double2* __restrict__ chirp, const double2* __restrict__ bh,
                                                  const double2* __restrict__ rtw, const double2* __restrict__ tw16k,
                                                  const double2* __restrict__ samples, double2* __restrict__ R) {
  using C = RegConv<32, 32>;
  const int n = 2 * k + 1;
  const int nwarps = blockDim.x >> 5, gmax = nwarps >> 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, pair = warp >> 1, half = warp & 1;
  double2* tw = sm;
  double2* cs = sm + C::RS;
  double2* ys = sm + C::RS + 1024;
  for (int i = threadIdx.x; i < C::RS; i += blockDim.x) tw[i] = __ldg(rtw + reg_rtw_offset(1024) + i);
  for (int i = threadIdx.x; i < n; i += blockDim.x) cs[i] = __ldg(chirp + i);
  double2* YA = ys + C::RS * (2 * pair);
  double2* YB = ys + C::RS * (2 * pair + 1);
  double2* Y = half ? YB : YA;
  const double2* H = bh + half * 1024;  // forward-direction kernel spectrum, even / odd bins
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  const double scale = OSPH_TWO_PI / (double)n;
  __syncthreads();
  for (int b0 = b_first; b0 < b_last; b0 += gmax) {
    const int Gr = min(gmax, b_last - b0);
    double2 v[32];
    {
      const double2* in = samples + (int64_t)(b0 + min(pair, Gr - 1)) * L * L + (int64_t)k * k;
#pragma unroll
      for (int n1 = 0; n1 < 32; ++n1) {
        const int t = n1 * 32 + lane;
        v[n1] = t < n ? cmul(__ldg(in + t), conj2(cs[t])) : make_double2(0.0, 0.0);
        if (half && t < n) v[n1] = cmul(v[n1], __ldg(tw16k + 8 * t));
      }
    }
    C::run<true>(v, Y, tw, H, lane);
    __syncwarp();
    if (half) {
#pragma unroll
      for (int n1 = 0; n1 < 32; ++n1) {
        const int t = n1 * 32 + lane;
        if (t < n) YB[t] = cmul(v[n1], conj2(__ldg(tw16k + 8 * t)));
      }
    }
    reg_pair_sync(pair);
    if (!half) {
#pragma unroll
      for (int n1 = 0; n1 < 32; ++n1) {
        const int t = n1 * 32 + lane;
        if (t < n) {
          const double2 x = cmul(cadd(v[n1], YB[t]), conj2(cs[t]));
          YA[t] = make_double2(scale * x.x, scale * x.y);
        }
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < Gr * (k + 1); idx += blockDim.x) {  // map-fastest writes of R
      const int gg = idx % Gr, m = idx / Gr;
      const double2* X = ys + C::RS * (2 * gg);
      const int64_t base = r_index(packed_pos(L, m, k - m), 0, b0 + gg, lgG, npos);
      R[base] = X[m];
      R[base + (1 << lgG)] = m == 0 ? make_double2(0.0, 0.0) : X[n - m];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(REG_THREADS, 2) k_ring_inverse_reg(
    int L, int B, int maps_per_block, const int* __restrict__ rings, const int* __restrict__ fft_n,
    const int64_t* __restrict__ chirp_off, const int64_t* __restrict__ bhat_off, const double2* __restrict__ chirp_all,
    const double2* __restrict__ bhat_all, const double2* __restrict__ rtw, const double* __restrict__ G,
    double2* __restrict__ samples) {
  extern __shared__ double2 sm[];
  const int k = rings[blockIdx.x];
  const int N = fft_n[k];
  const double2* chirp = chirp_all + chirp_off[k];
  const double2* bh = bhat_all + bhat_off[k] + N;  // inverse-direction kernel, natural order
  const int b_first = blockIdx.y * maps_per_block;
  const int b_last = min(B, b_first + maps_per_block);
  if (N == 1024) ring_inverse_reg<32, 32>(L, B, k, b_first, b_last, sm, chirp, bh, rtw, G, samples);
  else if (N == 512) ring_inverse_reg<32, 16>(L, B, k, b_first, b_last, sm, chirp, bh, rtw, G, samples);
  else ring_inverse_reg<16, 16>(L, B, k, b_first, b_last, sm, chirp, bh, rtw, G, samples);
}

template <int N1, int N2>
__device__ __forceinline__ void ring_forward_reg(int L, int k, int b_first, int b_last, int lgG, double2* sm,
                                                 const double2* __restrict__ chirp, const double2* __restrict__ bh,
                                                 const double2* __restrict__ rtw, const double2* __restrict__ samples,
                                                 double2* __restrict__ R) {
  using C = RegConv<N1, N2>;
  constexpr int GPW = 32 / C::T;
  const int n = 2 * k + 1;
  const int nwarps = blockDim.x >> 5;
  const int gmax = nwarps * GPW;
  const double2* tw = sm;
  const double2* hs = sm + C::RS;
  const double2* cs = sm + C::RS + C::N;
  double2* ys = reg_stage_tables<N1, N2>(sm, n, chirp, bh, rtw);
  const int lane = threadIdx.x & 31, g = (threadIdx.x >> 5) * GPW + lane / C::T, tid = lane % C::T;
  double2* Y = ys + C::RS * g;
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  const double scale = OSPH_TWO_PI / (double)n;
  __syncthreads();
  for (int b0 = b_first; b0 < b_last; b0 += gmax) {
    const int Gr = min(gmax, b_last - b0);
    double2 v[N1];
    {
      const double2* in = samples + (int64_t)(b0 + min(g, Gr - 1)) * L * L + (int64_t)k * k;
#pragma unroll
      for (int n1 = 0; n1 < N1 / 2; ++n1) {  // contiguous ring reads per map
        const int t = n1 * N2 + tid;
        v[n1] = t < n ? cmul(__ldg(in + t), conj2(cs[t])) : make_double2(0.0, 0.0);
      }
    }
    C::run(v, Y, tw, hs, tid);
    __syncwarp();  // every lane has re-read Y before the spectrum overwrites it
#pragma unroll
    for (int n1 = 0; n1 < N1 / 2; ++n1) {
      const int t = n1 * N2 + tid;
      if (t < n) {
        const double2 x = cmul(v[n1], conj2(cs[t]));
        Y[t] = make_double2(scale * x.x, scale * x.y);
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < Gr * (k + 1); idx += blockDim.x) {  // map-fastest writes of R
      const int gg = idx % Gr, m = idx / Gr;
      const double2* X = ys + C::RS * gg;
      const int64_t base = r_index(packed_pos(L, m, k - m), 0, b0 + gg, lgG, npos);
      R[base] = X[m];
      // order 0's - slot starts at zero and collects the sweep's -tone corrections that alias
      // to bin 0 (see scatter_rhs_multi)
      R[base + (1 << lgG)] = m == 0 ? make_double2(0.0, 0.0) : X[n - m];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(REG_THREADS, 2) k_ring_forward_reg(
    int L, int B, int maps_per_block, const int* __restrict__ rings, const int* __restrict__ fft_n,
    const int64_t* __restrict__ chirp_off, const int64_t* __restrict__ bhat_off, const double2* __restrict__ chirp_all,
    const double2* __restrict__ bhat_all, const double2* __restrict__ rtw, const double2* __restrict__ samples,
    double2* __restrict__ R, int bofs, int bend, int lgG) {
  extern __shared__ double2 sm[];
  const int k = rings[blockIdx.x];
  const int N = fft_n[k];
  const double2* chirp = chirp_all + chirp_off[k];
  const double2* bh = bhat_all + bhat_off[k];  // forward-direction kernel, natural order
  const int b_first = bofs + blockIdx.y * maps_per_block;
  const int b_last = min(bend, b_first + maps_per_block);
  if (N == 1024) ring_forward_reg<32, 32>(L, k, b_first, b_last, lgG, sm, chirp, bh, rtw, samples, R);
  else if (N == 512) ring_forward_reg<32, 16>(L, k, b_first, b_last, lgG, sm, chirp, bh, rtw, samples, R);
  else ring_forward_reg<16, 16>(L, k, b_first, b_last, lgG, sm, chirp, bh, rtw, samples, R);
}

// The 2048-point rings (their own launches: the code of the smaller classes stays lean).
__global__ void __launch_bounds__(REG_THREADS, 2) k_ring_inverse_reg2(
    int L, int B, int maps_per_block, const int* __restrict__ rings, const int64_t* __restrict__ chirp_off,
    const int64_t* __restrict__ bhat_off, const double2* __restrict__ chirp_all, const double2* __restrict__ bhat_all,
    const double2* __restrict__ rtw, const double2* __restrict__ tw16k, const double* __restrict__ G,
    double2* __restrict__ samples) {
  extern __shared__ double2 sm[];
  const int k = rings[blockIdx.x];
  const int b_first = blockIdx.y * maps_per_block;
  ring_inverse_reg2(L, B, k, b_first, min(B, b_first + maps_per_block), sm, chirp_all + chirp_off[k],
                    bhat_all + bhat_off[k] + 2048, rtw, tw16k, G, samples);
}

__global__ void __launch_bounds__(REG_THREADS, 2) k_ring_forward_reg2(
    int L, int B, int maps_per_block, const int* __restrict__ rings, const int64_t* __restrict__ chirp_off,
    const int64_t* __restrict__ bhat_off, const double2* __restrict__ chirp_all, const double2* __restrict__ bhat_all,
    const double2* __restrict__ rtw, const double2* __restrict__ tw16k, const double2* __restrict__ samples,
    double2* __restrict__ R, int bofs, int bend, int lgG) {
  extern __shared__ double2 sm[];
  const int k = rings[blockIdx.x];
  const int b_first = bofs + blockIdx.y * maps_per_block;
  ring_forward_reg2(L, k, b_first, min(bend, b_first + maps_per_block), lgG, sm, chirp_all + chirp_off[k],
                    bhat_all + bhat_off[k], rtw, tw16k, samples, R);
}

// launch shape of the register-resident kernels: warps per block, maps per block, shared memory
struct RegShape {
  int threads, mpb;
  size_t smem;
};
static RegShape reg_shape(int B, int nrings) {
  int warps = REG_WARPS;
  while (warps > 2 && (warps - 2) * 2 >= B) warps -= 2;  // small batches: fewer idle warps; even (2048-class warp pairs)
  // twiddles, kernel spectrum, chirp + one exchange matrix per group; 512- and 256-point rings
  // run two groups per warp
  const size_t ent = std::max<size_t>((size_t)RegConv<32, 32>::RS * (1 + warps) + 1536,
                                      (size_t)RegConv<32, 16>::RS * (1 + 2 * warps) + 768);
  static const int waves = getenv("OSPH_RING_WAVES") ? atoi(getenv("OSPH_RING_WAVES")) : 4;
  int mpb = 2 * warps;  // maps per block iteration of the half-warp classes
  while (mpb < B && (int64_t)nrings * ((B + mpb - 1) / mpb) > (int64_t)148 * 2 * waves) mpb *= 2;
  return {warps * 32, mpb, ent * sizeof(double2)};
}

// ---------------------------------------------------------------------------
// Rings whose Bluestein FFT is N = 2M = 16384 points (n = 2k+1 > 4096, L > 2048):
// one 2-CTA cluster per ring, each CTA holding M points.  Because n <= M the
// upper half of the chirped input is zero, so the first (span-M) stage of the
// decimation-in-frequency transform is local: CTA 0 keeps a_t, CTA 1 takes
// a_t W_N^t; each then runs an M-point DIF, multiplies by its half of the
// bit-reversed kernel spectrum and runs an M-point DIT -- exactly the first
// log2(N) - 1 stages of the N-point inverse.  Only outputs t < n <= M are
// needed, so the last (span-M) stage reduces to y_t = u_t + conj(W_N^t) v_t:
// CTA 1 applies the twiddle, CTA 0 adds CTA 1's half through distributed
// shared memory.  tw[t] = W_16384^t (the plan's twiddle table).
#define BIG_M 8192
#define BIG_LOGM 13

__device__ __forceinline__ void big_first_stage(double2* xs, int rank, int n, const double2* __restrict__ tw) {
  if (rank == 1)
    for (int t = threadIdx.x; t < n; t += blockDim.x) xs[fsw(t)] = cmul(xs[fsw(t)], __ldg(tw + t));
}

__device__ __forceinline__ void big_last_stage_prep(double2* xs, int rank, int n, const double2* __restrict__ tw) {
  if (rank == 1)
    for (int t = threadIdx.x; t < n; t += blockDim.x) xs[fsw(t)] = cmul(xs[fsw(t)], conj2(__ldg(tw + t)));
}

__global__ void __launch_bounds__(RING_THREADS) k_ring_inverse_bluestein2(
    int L, int B, int maps_per_block, const int* __restrict__ rings, const int64_t* __restrict__ chirp_off,
    const int64_t* __restrict__ bhat_off, const double2* __restrict__ chirp_all, const double2* __restrict__ bhat_all,
    const double2* __restrict__ tw, const double2* __restrict__ gsw, const double* __restrict__ G,
    double2* __restrict__ samples) {
  extern __shared__ double2 sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int k = rings[blockIdx.x >> 1];
  const int n = 2 * k + 1;
  double2* xs = sm + OSPH_SW_SMEM;
  load_stage_twiddles_smem(sm, BIG_LOGM, gsw);
  const StageTw twn{sm, gsw};
  const double2* xr = cl.map_shared_rank(xs, 1);
  const double2* chirp = chirp_all + chirp_off[k];
  const double2* bh = bhat_all + bhat_off[k] + 2 * BIG_M + rank * BIG_M;  // inverse-direction kernel, own half
  const int b_first = blockIdx.y * maps_per_block;
  const int b_last = min(B, b_first + maps_per_block);
  for (int b = b_first; b < b_last; ++b) {
    for (int t = threadIdx.x; t < BIG_M; t += blockDim.x) {
      double2 v = make_double2(0.0, 0.0);
      if (t < n) v = cmul(fold_bin(G, L, B, k, n, b, t), __ldg(chirp + t));
      xs[fsw(t)] = v;
    }
    __syncthreads();
    big_first_stage(xs, rank, n, tw);
    bluestein_convolve(xs, BIG_LOGM, 1, twn, bh);
    big_last_stage_prep(xs, rank, n, tw);
    cl.sync();
    if (rank == 0)
      for (int j = threadIdx.x; j < n; j += blockDim.x)
        samples[(int64_t)b * L * L + (int64_t)k * k + j] = cmul(cadd(xs[fsw(j)], xr[fsw(j)]), __ldg(chirp + j));
    cl.sync();  // CTA 1's half stays valid until CTA 0 has read it
  }
}

__global__ void __launch_bounds__(RING_THREADS) k_ring_forward_bluestein2(
    int L, int B, int maps_per_block, const int* __restrict__ rings, const int64_t* __restrict__ chirp_off,
    const int64_t* __restrict__ bhat_off, const double2* __restrict__ chirp_all, const double2* __restrict__ bhat_all,
    const double2* __restrict__ tw, const double2* __restrict__ gsw, const double2* __restrict__ samples,
    double2* __restrict__ R, int bofs, int bend, int lgG) {
  extern __shared__ double2 sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int k = rings[blockIdx.x >> 1];
  const int n = 2 * k + 1;
  double2* xs = sm + OSPH_SW_SMEM;
  load_stage_twiddles_smem(sm, BIG_LOGM, gsw);
  const StageTw twn{sm, gsw};
  const double2* xr = cl.map_shared_rank(xs, 1);
  const double2* chirp = chirp_all + chirp_off[k];
  const double2* bh = bhat_all + bhat_off[k] + rank * BIG_M;  // forward-direction kernel, own half
  const int b_first = bofs + blockIdx.y * maps_per_block;
  const int b_last = min(bend, b_first + maps_per_block);
  for (int b = b_first; b < b_last; ++b) {
    for (int t = threadIdx.x; t < BIG_M; t += blockDim.x) {
      double2 v = make_double2(0.0, 0.0);
      if (t < n) v = cmul(__ldg(samples + (int64_t)b * L * L + (int64_t)k * k + t), conj2(__ldg(chirp + t)));
      xs[fsw(t)] = v;
    }
    __syncthreads();
    big_first_stage(xs, rank, n, tw);
    bluestein_convolve(xs, BIG_LOGM, 1, twn, bh);
    big_last_stage_prep(xs, rank, n, tw);
    cl.sync();
    if (rank == 0)
      for (int t = threadIdx.x; t < n; t += blockDim.x)
        xs[fsw(t)] = cmul(cadd(xs[fsw(t)], xr[fsw(t)]), conj2(__ldg(chirp + t)));
    cl.sync();  // CTA 1 may overwrite its half only after CTA 0 has read it
    if (rank == 0) {
      scatter_rhs_multi<true>(xs, BIG_LOGM, L, lgG, k, n, b, 1, R);
      __syncthreads();
    }
  }
}

static size_t big_smem() { return sizeof(double2) * (size_t)(OSPH_SW_SMEM + BIG_M); }

static cudaError_t launch_big(const void* kern, osph_plan* p, int nb, int nbig, void** args) {
  const size_t smem = big_smem();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int mpb = maps_per_block_for(nb, nbig);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(2 * nbig), (unsigned)((nb + mpb - 1) / mpb));
  lc.blockDim = dim3(RING_THREADS);
  lc.dynamicSmemBytes = smem;
  lc.stream = p->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  *(int*)args[2] = mpb;
  e = cudaLaunchKernelExC(&lc, kern, args);
  p->launches++;
  return e;
}

static int max_fft(const osph_plan* p) {  // largest single-CTA Bluestein FFT
  int N = 0;
  for (int v : p->h_fft_n) N = (v > N && v <= OSPH_FFT_MAX) ? v : N;
  return N;
}

// maps per block: enough blocks for ~16 waves on 148 SMs (OSPH_RING_WAVES), at least 1
static int maps_per_block_for(int B, int rings) {
  static const int waves = getenv("OSPH_RING_WAVES") ? atoi(getenv("OSPH_RING_WAVES")) : 16;
  int mpb = B;
  while (mpb > 1 && (int64_t)rings * ((B + mpb - 1) / mpb) < 148 * waves) mpb = (mpb + 1) / 2;
  return mpb;
}

static size_t ring_smem(const osph_plan* p) {
  static const size_t budget = getenv("OSPH_RING_SMEM_KB") ? (size_t)atoi(getenv("OSPH_RING_SMEM_KB")) * 1024
                                                            : (size_t)RING_SMEM_BUDGET;
  const size_t need = sizeof(double2) * ((size_t)max_fft(p) + OSPH_SW_SMEM);
  return need > budget ? need : budget;
}

// The rings of the plan's inverse set (every ring, or a chain shard's range).
cudaError_t launch_ring_inverse(osph_plan* p, int B, double2* samples) {
  const int L = p->L;
  if (p->inv_n_big > 0) {  // the largest rings come first in d_inv_bluestein
    int Li = L, Bi = B, mpb = 0;
    const int* rings = p->d_inv_bluestein;
    void* args[] = {&Li, &Bi, &mpb, &rings, &p->d_chirp_off, &p->d_bhat_off, &p->d_chirp, &p->d_bhat,
                    &p->d_tw, &p->d_sw, &p->d_g, &samples};
    cudaError_t e = launch_big((const void*)k_ring_inverse_bluestein2, p, B, p->inv_n_big, args);
    if (e != cudaSuccess) return e;
  }
  if (p->inv_n_reg2 > 0) {  // 2048-point rings: the first inv_n_reg2 of the register-resident ones
    const RegShape sh = reg_shape(B, p->inv_n_reg2);
    cudaFuncSetAttribute(k_ring_inverse_reg2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.smem);
    dim3 grid(p->inv_n_reg2, (B + sh.mpb - 1) / sh.mpb);
    k_ring_inverse_reg2<<<grid, sh.threads, sh.smem, p->stream>>>(
        L, B, sh.mpb, p->d_inv_bluestein + (p->inv_n_bluestein - p->inv_n_reg), p->d_chirp_off, p->d_bhat_off,
        p->d_chirp, p->d_bhat, p->d_rtw, p->d_tw, p->d_g, samples);
    p->launches++;
  }
  if (p->inv_n_reg - p->inv_n_reg2 > 0) {
    const int nr = p->inv_n_reg - p->inv_n_reg2;
    const RegShape sh = reg_shape(B, nr);
    cudaFuncSetAttribute(k_ring_inverse_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.smem);
    dim3 grid(nr, (B + sh.mpb - 1) / sh.mpb);
    k_ring_inverse_reg<<<grid, sh.threads, sh.smem, p->stream>>>(
        L, B, sh.mpb, p->d_inv_bluestein + (p->inv_n_bluestein - nr), p->d_fft_n, p->d_chirp_off,
        p->d_bhat_off, p->d_chirp, p->d_bhat, p->d_rtw, p->d_g, samples);
    p->launches++;
  }
  const int nsmall = p->inv_n_bluestein - p->inv_n_big - p->inv_n_reg;
  if (nsmall > 0) {
    const int mpb = maps_per_block_for(B, nsmall);
    const size_t smem = ring_smem(p);
    cudaFuncSetAttribute(k_ring_inverse_bluestein, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(nsmall, (B + mpb - 1) / mpb);
    k_ring_inverse_bluestein<<<grid, RING_THREADS, smem, p->stream>>>(
        L, B, mpb, p->d_inv_bluestein + p->inv_n_big, p->d_fft_n, p->d_chirp_off, p->d_bhat_off, p->d_chirp,
        p->d_bhat, p->d_sw, p->d_g, samples, (int)(smem / sizeof(double2)));
    p->launches++;
  }
  const int ndirect = p->inv_direct_hi - p->inv_direct_lo;
  if (ndirect > 0) {
    const int mpb = maps_per_block_for(B, ndirect);
    dim3 grid(ndirect, (B + mpb - 1) / mpb);
    k_ring_inverse_direct<<<grid, 128, 0, p->stream>>>(L, B, mpb, p->inv_direct_lo, p->d_roots, p->d_g, samples);
    p->launches++;
  }
  return cudaGetLastError();
}

cudaError_t launch_ring_forward(osph_plan* p, int B, const double2* samples, int bofs, int nb, bool plain) {
  const int L = p->L;
  if (nb < 0) nb = B;
  int lgG = plain ? 0 : __builtin_ctz(sweep_maps_per_team(p, B));  // team-major R (common.cuh)
  if (p->n_big_rings > 0) {
    int Li = L, Bi = B, mpb = 0, b0 = bofs, b1 = bofs + nb;
    const int* rings = p->d_bluestein_rings;
    void* args[] = {&Li, &Bi, &mpb, &rings, &p->d_chirp_off, &p->d_bhat_off, &p->d_chirp, &p->d_bhat,
                    &p->d_tw, &p->d_sw, &samples, &p->d_r, &b0, &b1, &lgG};
    cudaError_t e = launch_big((const void*)k_ring_forward_bluestein2, p, nb, p->n_big_rings, args);
    if (e != cudaSuccess) return e;
  }
  if (p->n_reg2_rings > 0) {  // 2048-point rings: the first n_reg2_rings of the register-resident ones
    const RegShape sh = reg_shape(nb, p->n_reg2_rings);
    cudaFuncSetAttribute(k_ring_forward_reg2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.smem);
    dim3 grid(p->n_reg2_rings, (nb + sh.mpb - 1) / sh.mpb);
    k_ring_forward_reg2<<<grid, sh.threads, sh.smem, p->stream>>>(
        L, B, sh.mpb, p->d_bluestein_rings + (p->n_bluestein_rings - p->n_reg_rings), p->d_chirp_off, p->d_bhat_off,
        p->d_chirp, p->d_bhat, p->d_rtw, p->d_tw, samples, p->d_r, bofs, bofs + nb, lgG);
    p->launches++;
  }
  if (p->n_reg_rings - p->n_reg2_rings > 0) {
    const int nr = p->n_reg_rings - p->n_reg2_rings;
    const RegShape sh = reg_shape(nb, nr);
    cudaFuncSetAttribute(k_ring_forward_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.smem);
    dim3 grid(nr, (nb + sh.mpb - 1) / sh.mpb);
    k_ring_forward_reg<<<grid, sh.threads, sh.smem, p->stream>>>(
        L, B, sh.mpb, p->d_bluestein_rings + (p->n_bluestein_rings - nr), p->d_fft_n, p->d_chirp_off,
        p->d_bhat_off, p->d_chirp, p->d_bhat, p->d_rtw, samples, p->d_r, bofs, bofs + nb, lgG);
    p->launches++;
  }
  const int nsmall = p->n_bluestein_rings - p->n_big_rings - p->n_reg_rings;
  if (nsmall > 0) {
    const int mpb = maps_per_block_for(nb, nsmall);
    const size_t smem = ring_smem(p);
    cudaFuncSetAttribute(k_ring_forward_bluestein, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(nsmall, (nb + mpb - 1) / mpb);
    k_ring_forward_bluestein<<<grid, RING_THREADS, smem, p->stream>>>(
        L, B, mpb, p->d_bluestein_rings + p->n_big_rings, p->d_fft_n, p->d_chirp_off, p->d_bhat_off, p->d_chirp,
        p->d_bhat, p->d_sw, samples, p->d_r, (int)(smem / sizeof(double2)), bofs, bofs + nb, lgG);
    p->launches++;
  }
  if (p->n_direct_rings > 0) {
    const int mpb = maps_per_block_for(nb, p->n_direct_rings);
    dim3 grid(p->n_direct_rings, (nb + mpb - 1) / mpb);
    k_ring_forward_direct<<<grid, 128, 0, p->stream>>>(L, B, mpb, p->d_roots, samples, p->d_r, bofs, bofs + nb, lgG);
    p->launches++;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Single-ring two-bin analysis, the public ring_analysis helper
// (transform.py:115-131): delta * sum_j v_j e^{-+ 2 pi i m j / n}.
__global__ void k_ring_pair(int n, int m, const double2* __restrict__ v, double2* __restrict__ out) {
  __shared__ double red[4][32];
  double pr = 0.0, pi = 0.0, nr = 0.0, ni = 0.0;
  const int step = ((m % n) + n) % n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int r = (int)(((int64_t)j * step) % n);
    double s, c;
    sincospi(2.0 * (double)r / (double)n, &s, &c);
    const double2 x = v[j];
    pr += x.x * c + x.y * s;  // x * conj(w)
    pi += x.y * c - x.x * s;
    nr += x.x * c - x.y * s;  // x * w
    ni += x.y * c + x.x * s;
  }
  for (int o = 16; o > 0; o >>= 1) {
    pr += __shfl_xor_sync(0xffffffffu, pr, o);
    pi += __shfl_xor_sync(0xffffffffu, pi, o);
    nr += __shfl_xor_sync(0xffffffffu, nr, o);
    ni += __shfl_xor_sync(0xffffffffu, ni, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = pr;
    red[1][w] = pi;
    red[2][w] = nr;
    red[3][w] = ni;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a[4] = {0, 0, 0, 0};
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
      for (int t = 0; t < 4; ++t) a[t] += red[t][q];
    const double delta = OSPH_TWO_PI / (double)n;
    out[0] = make_double2(delta * a[0], delta * a[1]);
    out[1] = make_double2(delta * a[2], delta * a[3]);
  }
}

cudaError_t launch_ring_pair(int n, int m, const double2* v, double2* out, cudaStream_t st) {
  k_ring_pair<<<1, 256, 0, st>>>(n, m, v, out);
  return cudaGetLastError();
}
