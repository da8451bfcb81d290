// EXPERIMENTAL, NOT BUILT: warp-level four-step Bluestein ring DFTs (k_ring_*_wfft).
// Measured slower than the block-level kernels at config 2 (ring inverse 0.45 vs
// 0.37 ms; 255 registers, 8 warps per SM), see DESIGN.md section 11.
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
#include <vector>

#include "fft.cuh"
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


// ---------------------------------------------------------------------------
// Warp-level Bluestein ring DFTs for FFT sizes N = 32 * N2, N2 in {8, 16, 32}
// (rings 33 <= k <= 511).  One warp convolves G = 32 / N2 maps of a ring at a
// time (G * N = 1024 points, 32 complex values per lane in registers); the
// power-of-two FFT is a four-step FFT (N = 32 x N2):
//   lane (g, j2): a[N2 j1 + j2], j1 = 0..31 -> 32-point DFT over j1 (registers)
//                 -> twiddle W_N^{j2 k1} -> shared-memory transpose (per warp)
//   lane k1:      N2-point DFTs over j2 (G of them) -> A[k1 + 32 k2]
// then the product with the kernel spectrum and the same steps backwards,
// so a whole Bluestein convolution takes two warp-private transposes and
// __syncwarp instead of 2 log4(N) block-wide barrier passes.

// e^{-2 pi i k / 32}, k < 16 (compile-time k after unrolling)
__device__ __forceinline__ double2 wf_w32(int k) {
  switch (k) {
    case 0: return make_double2(1.0, 0.0);
    case 1: return make_double2(0.9807852804032304, -0.19509032201612825);
    case 2: return make_double2(0.9238795325112867, -0.3826834323650898);
    case 3: return make_double2(0.8314696123025452, -0.5555702330196022);
    case 4: return make_double2(0.7071067811865476, -0.7071067811865475);
    case 5: return make_double2(0.5555702330196023, -0.8314696123025452);
    case 6: return make_double2(0.38268343236508984, -0.9238795325112867);
    case 7: return make_double2(0.19509032201612833, -0.9807852804032304);
    case 8: return make_double2(0.0, -1.0);
    case 9: return make_double2(-0.1950903220161282, -0.9807852804032304);
    case 10: return make_double2(-0.3826834323650897, -0.9238795325112867);
    case 11: return make_double2(-0.555570233019602, -0.8314696123025455);
    case 12: return make_double2(-0.7071067811865475, -0.7071067811865476);
    case 13: return make_double2(-0.8314696123025453, -0.5555702330196022);
    case 14: return make_double2(-0.9238795325112867, -0.3826834323650899);
    case 15: return make_double2(-0.9807852804032304, -0.1950903220161286);
    default: return make_double2(1.0, 0.0);
  }
}

// In-register radix-2 FFT of M points v[OFF + i], natural order in and out
// (DIT after a compile-time bit reversal of the register names).
template <int M>
__device__ __forceinline__ constexpr int wf_brev(int x) {
  int r = 0;
  for (int i = 1; i < M; i <<= 1) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r;
}
template <int M, int OFF, bool INV>
__device__ __forceinline__ void wf_reg_fft(double2 (&v)[32]) {
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const int j = wf_brev<M>(i);
    if (j > i) {
      const double2 t = v[OFF + i];
      v[OFF + i] = v[OFF + j];
      v[OFF + j] = t;
    }
  }
#pragma unroll
  for (int h = 1; h < M; h <<= 1) {
#pragma unroll
    for (int s = 0; s < M; s += 2 * h) {
#pragma unroll
      for (int p = 0; p < h; ++p) {
        const double2 a = v[OFF + s + p];
        double2 b = v[OFF + s + p + h];
        if (p != 0) {
          double2 w = wf_w32(p * (32 / (2 * h)));  // W_{2h}^p
          if (INV) w.y = -w.y;
          b = cmul(w, b);
        }
        v[OFF + s + p] = cadd(a, b);
        v[OFF + s + p + h] = csub(a, b);
      }
    }
  }
}

// The G groups of N2 registers: v[gg * N2 .. gg * N2 + N2), gg < G, each transformed.
template <int N2, int G, bool INV, int GG = 0>
__device__ __forceinline__ void wf_group_ffts(double2 (&v)[32]) {
  if constexpr (GG < G) {
    wf_reg_fft<N2, GG * N2, INV>(v);
    wf_group_ffts<N2, G, INV, GG + 1>(v);
  }
}

// W_N^e (forward sign) from the plan's table tw[j] = e^{-2 pi i j / 16384}, j < 8192.
__device__ __forceinline__ double2 wf_twiddle(const double2* __restrict__ tw, int e, int logN) {
  const int half = 1 << (logN - 1);
  const int sh = 14 - logN;
  if (e < half) return __ldg(tw + (e << sh));
  const double2 w = __ldg(tw + ((e - half) << sh));
  return make_double2(-w.x, -w.y);
}

// v[k1] *= W_N^{(+-) j2 k1}, k1 < 32: the table at k1 = 0, 8, 16, 24 and a
// step of W_N^{j2} in between (at most 7 products: ~1e-15 relative, far below
// the transform's tolerance), so only five twiddles are loaded per lane.
template <int LOGN, bool CONJ>
__device__ __forceinline__ void wf_twiddle_rows(double2 (&v)[32], const double2* __restrict__ tw, int j2) {
  double2 st = wf_twiddle(tw, j2, LOGN);
  if (CONJ) st = conj2(st);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double2 w = wf_twiddle(tw, j2 * 8 * q, LOGN);
    if (CONJ) w = conj2(w);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (q > 0 || r > 0) v[8 * q + r] = cmul(v[8 * q + r], w);
      if (r < 7) w = cmul(w, st);
    }
  }
}

// The Bluestein convolution of the warp's G maps, in place: on entry lane
// (g, j2) = (lane / N2, lane % N2) holds a[N2 j1 + j2] in v[j1]; on exit it
// holds y[N2 j1 + j2] = (a (*) b)[.] (circular convolution with the kernel
// whose spectrum / N is bh_br, stored bit-reversed).  S: the warp's shared
// scratch of G * 32 * (N2 + 1) complex.
template <int LOGN2>
__device__ __forceinline__ void wf_convolve(double2 (&v)[32], double2* S, const double2* __restrict__ bh_br,
                                            const double2* __restrict__ tw, int lane) {
  constexpr int N2 = 1 << LOGN2, G = 32 / N2, LOGN = 5 + LOGN2, LD = N2 + 1;
  const int g = lane >> LOGN2, j2 = lane & (N2 - 1);
  __syncwarp();  // the caller's reads of S are done
  wf_reg_fft<32, 0, false>(v);  // over j1 -> k1
  wf_twiddle_rows<LOGN, false>(v, tw, j2);
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) S[(g * 32 + k1) * LD + j2] = v[k1];
  __syncwarp();
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int jj = 0; jj < N2; ++jj) v[gg * N2 + jj] = S[(gg * 32 + lane) * LD + jj];
  // lane = k1 now: N2-point DFTs over j2 -> k2, product with the spectrum, back
  wf_group_ffts<N2, G, false>(v);
#pragma unroll
  for (int k2 = 0; k2 < N2; ++k2) {
    const int q = lane + 32 * k2;
    const double2 h = __ldg(bh_br + (__brev((unsigned)q) >> (32 - LOGN)));
#pragma unroll
    for (int gg = 0; gg < G; ++gg) v[gg * N2 + k2] = cmul(v[gg * N2 + k2], h);
  }
  wf_group_ffts<N2, G, true>(v);
  __syncwarp();  // every lane has read S
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int jj = 0; jj < N2; ++jj) S[(gg * 32 + lane) * LD + jj] = v[gg * N2 + jj];
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) v[k1] = S[(g * 32 + k1) * LD + j2];
  wf_twiddle_rows<LOGN, true>(v, tw, j2);
  wf_reg_fft<32, 0, true>(v);  // over k1 -> j1
  __syncwarp();  // every lane has read S
}

#define WF_WARPS 4
#define WF_MAPS 16  // maps per block: 4 per warp, G per pass

template <int LOGN2>
__global__ void __launch_bounds__(32 * WF_WARPS) k_ring_forward_wfft(
    int L, int B, const int* __restrict__ rings, const int64_t* __restrict__ chirp_off,
    const int64_t* __restrict__ bhat_off, const double2* __restrict__ chirp_all, const double2* __restrict__ bhat_all,
    const double2* __restrict__ tw, const double2* __restrict__ samples, double2* __restrict__ R, int bofs, int bend,
    int lgG) {
  constexpr int N2 = 1 << LOGN2, G = 32 / N2, LD = N2 + 1, N = 32 * N2, LOGN = 5 + LOGN2;
  extern __shared__ double2 wf_sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* S = wf_sm + (size_t)warp * G * 32 * LD;  // also the flat [g][t] staging of G * N values
  const int k = rings[blockIdx.x];
  const int n = 2 * k + 1;
  const double2* chirp = chirp_all + chirp_off[k];
  const double2* bh = bhat_all + bhat_off[k];  // forward-direction kernel
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  const double scale = OSPH_TWO_PI / (double)n;
  const int g = lane >> LOGN2, j2 = lane & (N2 - 1);
  const int bw = bofs + blockIdx.y * WF_MAPS + warp * (WF_MAPS / WF_WARPS);
#pragma unroll 1
  for (int pass = 0; pass < (WF_MAPS / WF_WARPS + G - 1) / G; ++pass) {
    const int b0 = bw + pass * G;
    if (b0 >= bend) break;  // warp-uniform
    // ring samples of the pass's maps, coalesced, times conj(chirp) -> S[g][t]
#pragma unroll 1
    for (int idx = lane; idx < G * N; idx += 32) {
      const int gg = idx >> LOGN, t = idx & (N - 1);
      const int b = b0 + gg;
      double2 a = make_double2(0.0, 0.0);
      if (t < n && b < bend && pass * G + gg < WF_MAPS / WF_WARPS)
        a = cmul(__ldg(samples + (int64_t)b * L * L + (int64_t)k * k + t), conj2(__ldg(chirp + t)));
      S[idx] = a;
    }
    __syncwarp();
    double2 v[32];
#pragma unroll
    for (int j1 = 0; j1 < 32; ++j1) v[j1] = S[g * N + N2 * j1 + j2];
    wf_convolve<LOGN2>(v, S, bh, tw, lane);
#pragma unroll
    for (int j1 = 0; j1 < 32; ++j1) S[g * N + N2 * j1 + j2] = v[j1];
    __syncwarp();
    // bins -> right-hand sides: bin t is the + tone of order m = t (t <= k) or the
    // - tone of order m = n - t (t > k)
#pragma unroll 1
    for (int idx = lane; idx < G * n; idx += 32) {
      const int gg = idx / n, t = idx - gg * n;
      const int b = b0 + gg;
      if (b >= bend || pass * G + gg >= WF_MAPS / WF_WARPS) continue;
      const double2 X = cmul(S[gg * N + t], conj2(__ldg(chirp + t)));
      const int m = t <= k ? t : n - t;
      const int64_t base = r_index(packed_pos(L, m, k - m), t <= k ? 0 : 1, b, lgG, npos);
      R[base] = make_double2(scale * X.x, scale * X.y);
      if (t == 0) R[base + (1 << lgG)] = make_double2(0.0, 0.0);  // order 0's - slot (sweep.cu)
    }
    __syncwarp();
  }
}

template <int LOGN2>
__global__ void __launch_bounds__(32 * WF_WARPS) k_ring_inverse_wfft(
    int L, int B, const int* __restrict__ rings, const int64_t* __restrict__ chirp_off,
    const int64_t* __restrict__ bhat_off, const double2* __restrict__ chirp_all, const double2* __restrict__ bhat_all,
    const double2* __restrict__ tw, const double* __restrict__ Gbuf, double2* __restrict__ samples) {
  constexpr int N2 = 1 << LOGN2, G = 32 / N2, LD = N2 + 1, N = 32 * N2;
  extern __shared__ double2 wf_sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* S = wf_sm + (size_t)warp * G * 32 * LD;
  const int k = rings[blockIdx.x];
  const int n = 2 * k + 1;
  const double2* chirp = chirp_all + chirp_off[k];
  const double2* bh = bhat_all + bhat_off[k] + N;  // inverse-direction kernel (second N entries)
  const int g = lane >> LOGN2, j2 = lane & (N2 - 1);
  const int bw = blockIdx.y * WF_MAPS + warp * (WF_MAPS / WF_WARPS);
#pragma unroll 1
  for (int pass = 0; pass < (WF_MAPS / WF_WARPS + G - 1) / G; ++pass) {
    const int b0 = bw + pass * G;
    if (b0 >= B) break;  // warp-uniform
    // fold the tones into the ring's bins (map-fastest reads of G), times the chirp -> S[g][t]
#pragma unroll 1
    for (int idx = lane; idx < G * N; idx += 32) {
      const int gg = idx & (G - 1), t = idx >> (5 - LOGN2);
      const int b = b0 + gg;
      double2 a = make_double2(0.0, 0.0);
      if (t < n && b < B && pass * G + gg < WF_MAPS / WF_WARPS)
        a = cmul(fold_bin(Gbuf, L, B, k, n, b, t), __ldg(chirp + t));
      S[gg * N + t] = a;
    }
    __syncwarp();
    double2 v[32];
#pragma unroll
    for (int j1 = 0; j1 < 32; ++j1) v[j1] = S[g * N + N2 * j1 + j2];
    wf_convolve<LOGN2>(v, S, bh, tw, lane);
#pragma unroll
    for (int j1 = 0; j1 < 32; ++j1) S[g * N + N2 * j1 + j2] = v[j1];
    __syncwarp();
#pragma unroll 1
    for (int idx = lane; idx < G * n; idx += 32) {  // contiguous ring writes per map
      const int gg = idx / n, t = idx - gg * n;
      const int b = b0 + gg;
      if (b >= B || pass * G + gg >= WF_MAPS / WF_WARPS) continue;
      samples[(int64_t)b * L * L + (int64_t)k * k + t] = cmul(S[gg * N + t], __ldg(chirp + t));
    }
    __syncwarp();
  }
}

static size_t wf_smem(int logn2) {
  const int n2 = 1 << logn2;
  return sizeof(double2) * (size_t)WF_WARPS * (32 / n2) * 32 * (n2 + 1);
}

// Rings [r0, r1) of a list sorted largest first whose FFT size is N = 32 << logn2.
static void wf_class(const std::vector<int>& list, const std::vector<int>& fft_n, int logn2, int& r0, int& r1) {
  const int N = 32 << logn2;
  r0 = r1 = (int)list.size();
  for (int i = 0; i < (int)list.size(); ++i)
    if (fft_n[list[i]] == N) {
      if (r0 == (int)list.size()) r0 = i;
      r1 = i + 1;
    }
}

// Count of the list's trailing rings the warp kernels take (N <= 1024).
static int wf_suffix(const std::vector<int>& list, const std::vector<int>& fft_n) {
  int c = 0;
  for (int i = (int)list.size() - 1; i >= 0 && fft_n[list[i]] >= 256 && fft_n[list[i]] <= 1024; --i) ++c;
  static const bool off = getenv("OSPH_RING_WFFT") && atoi(getenv("OSPH_RING_WFFT")) == 0;
  return off ? 0 : c;
}

template <int LOGN2>
static cudaError_t wf_launch_fwd(osph_plan* p, const int* d_list, const std::vector<int>& list, int B,
                                 const double2* samples, int bofs, int nb, int lgG) {
  int r0, r1;
  wf_class(list, p->h_fft_n, LOGN2, r0, r1);
  if (r1 <= r0) return cudaSuccess;
  const size_t smem = wf_smem(LOGN2);
  cudaError_t e = cudaFuncSetAttribute(k_ring_forward_wfft<LOGN2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(r1 - r0, (nb + WF_MAPS - 1) / WF_MAPS);
  k_ring_forward_wfft<LOGN2><<<grid, 32 * WF_WARPS, smem, p->stream>>>(
      p->L, B, d_list + r0, p->d_chirp_off, p->d_bhat_off, p->d_chirp, p->d_bhat, p->d_tw, samples, p->d_r, bofs,
      bofs + nb, lgG);
  p->launches++;
  return cudaGetLastError();
}

template <int LOGN2>
static cudaError_t wf_launch_inv(osph_plan* p, const int* d_list, const std::vector<int>& list, int B,
                                 double2* samples) {
  int r0, r1;
  wf_class(list, p->h_fft_n, LOGN2, r0, r1);
  if (r1 <= r0) return cudaSuccess;
  const size_t smem = wf_smem(LOGN2);
  cudaError_t e = cudaFuncSetAttribute(k_ring_inverse_wfft<LOGN2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(r1 - r0, (B + WF_MAPS - 1) / WF_MAPS);
  k_ring_inverse_wfft<LOGN2><<<grid, 32 * WF_WARPS, smem, p->stream>>>(
      p->L, B, d_list + r0, p->d_chirp_off, p->d_bhat_off, p->d_chirp, p->d_bhat, p->d_tw, p->d_g, samples);
  p->launches++;
  return cudaGetLastError();
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
  // rings with 256 <= N <= 1024 (the tail of the list): warp-level kernels
  const int nwf = wf_suffix(p->h_inv_bluestein, p->h_fft_n);
  if (nwf > 0) {
    cudaError_t e;
    if ((e = wf_launch_inv<5>(p, p->d_inv_bluestein, p->h_inv_bluestein, B, samples)) != cudaSuccess) return e;
    if ((e = wf_launch_inv<4>(p, p->d_inv_bluestein, p->h_inv_bluestein, B, samples)) != cudaSuccess) return e;
    if ((e = wf_launch_inv<3>(p, p->d_inv_bluestein, p->h_inv_bluestein, B, samples)) != cudaSuccess) return e;
  }
  const int nsmall = p->inv_n_bluestein - p->inv_n_big - nwf;
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

cudaError_t launch_ring_forward(osph_plan* p, int B, const double2* samples, int bofs, int nb) {
  const int L = p->L;
  if (nb < 0) nb = B;
  int lgG = __builtin_ctz(sweep_maps_per_team(p, B));  // team-major R (common.cuh)
  if (p->n_big_rings > 0) {
    int Li = L, Bi = B, mpb = 0, b0 = bofs, b1 = bofs + nb;
    const int* rings = p->d_bluestein_rings;
    void* args[] = {&Li, &Bi, &mpb, &rings, &p->d_chirp_off, &p->d_bhat_off, &p->d_chirp, &p->d_bhat,
                    &p->d_tw, &p->d_sw, &samples, &p->d_r, &b0, &b1, &lgG};
    cudaError_t e = launch_big((const void*)k_ring_forward_bluestein2, p, nb, p->n_big_rings, args);
    if (e != cudaSuccess) return e;
  }
  const int nwf = wf_suffix(p->h_bluestein_rings, p->h_fft_n);
  if (nwf > 0) {
    cudaError_t e;
    const int* dl = p->d_bluestein_rings;
    const std::vector<int>& hl = p->h_bluestein_rings;
    if ((e = wf_launch_fwd<5>(p, dl, hl, B, samples, bofs, nb, lgG)) != cudaSuccess) return e;
    if ((e = wf_launch_fwd<4>(p, dl, hl, B, samples, bofs, nb, lgG)) != cudaSuccess) return e;
    if ((e = wf_launch_fwd<3>(p, dl, hl, B, samples, bofs, nb, lgG)) != cudaSuccess) return e;
  }
  const int nsmall = p->n_bluestein_rings - p->n_big_rings - nwf;
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
