// tables.cu -- per-plan O(L^2) tables (data independent, built once per plan).
//
//  * recurrence factors a_lm = sqrt((l^2-m^2)/((2l-1)(2l+1))) and 1/a_(l+1)m,
//    packed order-major exactly like _packed_tables (transform.py:268-291);
//  * "start" table: for every (order m, ring k) the first degree ls whose
//    Y_lm(theta_k) is inside the double range, with the recurrence pair
//    (P_(ls-1), P_ls).  It is produced by the reference's rescaled upward
//    recurrence (legendre.py:64-96: window [2^-500, 2^500], shifts of 2^1000);
//    below ls every value is < 2^-500 and contributes nothing, so the hot
//    kernels start the plain recurrence at ls with no rescaling branches;
//  * Bluestein chirps and kernel spectra for the odd-length ring DFTs, and the
//    FFT twiddle table.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <numeric>

#include "fft.cuh"
#include "plan.cuh"

// a_lm and 1/a_(l+1)m for l = m..L-1, one block row per order.
__global__ void k_rec_table(int L, double2* __restrict__ rec) {
  const int m = blockIdx.y;
  const double mm = (double)m * (double)m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L - m; i += gridDim.x * blockDim.x) {
    const double l = (double)(m + i);
    const double a = sqrt((l * l - mm) / ((2.0 * l - 1.0) * (2.0 * l + 1.0)));
    const double l1 = l + 1.0;
    const double an = sqrt((l1 * l1 - mm) / ((2.0 * l1 - 1.0) * (2.0 * l1 + 1.0)));
    rec[packed_pos(L, m, i)] = make_double2(a, 1.0 / an);
  }
}

// Seeds Y_mm(theta_k) = (-1)^m sqrt((2m+1)/4pi) prod_{q<m} sin(theta) sqrt((2q+1)/(2q+2))
// (legendre.py:75-80, 134-136) as (mantissa, number of 2^-1000 shifts); one
// thread per ring walks m upward keeping the running product in the window.
__global__ void k_seeds(int L, const double* __restrict__ sinth, double* __restrict__ seed_mant,
                        int* __restrict__ seed_shift) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  const double s = sinth[k];
  double mant = 1.0;
  int j = 0;
  for (int m = 0; m < L; ++m) {
    double v = sqrt((2.0 * m + 1.0) / (4.0 * OSPH_PI)) * mant;
    int jj = j;
    if (fabs(v) < OSPH_TINY && v != 0.0) {
      v *= OSPH_UP;
      jj += 1;
    }
    seed_mant[(int64_t)m * L + k] = (m & 1) ? -v : v;
    seed_shift[(int64_t)m * L + k] = jj;
    const double q = (double)m;
    mant *= s * sqrt((2.0 * q + 1.0) / (2.0 * q + 2.0));
    if (fabs(mant) < OSPH_TINY && mant != 0.0) {
      mant *= OSPH_UP;
      j += 1;
    }
  }
}

// For each (m, k): run the rescaled recurrence from the seed until the value is
// back in the double range (shift count 0); record ls and the pair there.
__global__ void k_start_table(int L, const double* __restrict__ costh, const double2* __restrict__ rec,
                              const double* __restrict__ seed_mant, int* __restrict__ ls_tab,
                              double2* __restrict__ pstart) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (k >= L) return;
  const int64_t t = (int64_t)m * L + k;
  int j = ls_tab[t];  // holds the seed shift count on entry
  double curr = seed_mant[t];
  double prev = 0.0;
  int ls = m;
  if (j > 0) {
    const double c = costh[k];
    const double2* rm = rec + packed_pos(L, m, 0);
    ls = L;
    for (int l = m; l < L - 1; ++l) {
      const double2 ar = rm[l - m];
      const double nxt = (c * curr - ar.x * prev) * ar.y;
      prev = curr;
      curr = nxt;
      const double ac = fabs(curr);
      if (ac > OSPH_BIG) {
        curr *= OSPH_DOWN;
        prev *= OSPH_DOWN;
        j -= 1;
      } else if (ac < OSPH_TINY && fabs(prev) < OSPH_TINY && (curr != 0.0 || prev != 0.0)) {
        curr *= OSPH_UP;
        prev *= OSPH_UP;
        j += 1;
      }
      if (j == 0) {
        ls = l + 1;
        break;
      }
    }
  }
  ls_tab[t] = ls;
  pstart[t] = make_double2(prev, curr);
}

// legendre_table(m, thetas, L) (legendre.py:110-143) for every plan ring k:
// out[(l - m) * ld + k] = Y_lm(theta_k, 0), l = m..L-1 (degree-major, so the
// stores of a warp are coalesced).  Degrees below the start degree ls are
// < 2^-500 (the reference's rescaled values there are below every term they
// are summed with) and are written as 0; from ls on, the plain recurrence in
// the same fma form as the hot kernels.
__global__ void k_legendre_block(int L, int m, const double* __restrict__ costh, const double2* __restrict__ rec,
                                 const int* __restrict__ ls_tab, const double2* __restrict__ pstart,
                                 double* __restrict__ out, int64_t ld) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  const int64_t t = (int64_t)m * L + k;
  const int ls = ls_tab[t];
  for (int l = m; l < min(ls, L); ++l) out[(int64_t)(l - m) * ld + k] = 0.0;
  if (ls >= L) return;
  const double2 pr = pstart[t];
  const double x = costh[k];
  const double2* rm = rec + packed_pos(L, m, 0);
  double p0 = pr.x, p1 = pr.y;
  out[(int64_t)(ls - m) * ld + k] = p1;
  for (int l = ls; l < L - 1; ++l) {
    const double2 ar = rm[l - m];
    const double nxt = fma(x, p1, -ar.x * p0) * ar.y;
    p0 = p1;
    p1 = nxt;
    out[(int64_t)(l + 1 - m) * ld + k] = p1;
  }
}

cudaError_t launch_legendre_block(osph_plan* p, int m, double* out, int64_t ld) {
  k_legendre_block<<<(p->L + 127) / 128, 128, 0, p->stream>>>(p->L, m, p->d_cos, p->d_rec, p->d_ls, p->d_pstart,
                                                              out, ld);
  return cudaGetLastError();
}

__global__ void k_stage_twiddles(double2* __restrict__ sw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= OSPH_SW_GLOBAL / 2 - 1) return;  // i = (h - 1) + pos over h = 1, 2, 4, ..., 4096 (i < 8191)
  const int lh = 31 - __clz(i + 1);
  const int h = 1 << lh, pos = i + 1 - h;
  double s, c;
  sincospi(-2.0 * (double)pos / (double)(2 * h), &s, &c);
  sw[2 * (h - 1) + pos] = make_double2(c, s);
  sincospi(-2.0 * (double)pos / (double)(4 * h), &s, &c);
  sw[2 * (h - 1) + h + pos] = make_double2(c, s);
}

// Inter-pass twiddles of the register-resident convolutions (fft_reg.cuh):
// for N = N1 N2 the padded matrix TW[k1 (N2 + 1) + n2] = e^{-2 pi i k1 n2 / N}.
// Classes: 256 = 16 x 16 at 0, 512 = 32 x 16 at 272, 1024 = 32 x 32 at 816.
__global__ void k_reg_twiddles(double2* __restrict__ rtw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= OSPH_RTW_SIZE) return;
  int N1, N2, base;
  if (i < 272) {
    N1 = 16; N2 = 16; base = 0;
  } else if (i < 816) {
    N1 = 32; N2 = 16; base = 272;
  } else {
    N1 = 32; N2 = 32; base = 816;
  }
  const int r = i - base, k1 = r / (N2 + 1), n2 = r - k1 * (N2 + 1);
  double s = 0.0, c = 1.0;
  if (n2 < N2) sincospi(-2.0 * (double)(k1 * n2) / (double)(N1 * N2), &s, &c);
  rtw[i] = make_double2(c, s);
}

__global__ void k_twiddles(double2* __restrict__ tw) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= OSPH_TW_SIZE / 2) return;
  double s, c;
  sincospi(-2.0 * (double)j / (double)OSPH_TW_SIZE, &s, &c);
  tw[j] = make_double2(c, s);
}

// Direct-DFT rings: roots e^{2 pi i r/n} at k*k + r (transform.py:294-301).
__global__ void k_small_roots(int nrings, double2* __restrict__ roots) {
  const int k = blockIdx.x;
  if (k >= nrings) return;
  const int n = 2 * k + 1;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    double s, c;
    sincospi(2.0 * (double)r / (double)n, &s, &c);
    roots[(int64_t)k * k + r] = make_double2(c, s);
  }
}

// Bluestein tables for one ring per block: chirp[t] = e^{i pi t^2/n} and, for
// both directions, bhat = FFT_N(conjugate chirp kernel) / N.
// One block per ring (grid-stride over nrings).  scratch == nullptr: the
// N-point work array lives in shared memory; otherwise in global memory at
// scratch + blockIdx.x * N (the 16384-point kernels of L > 2048, one-time setup).
__global__ void k_bluestein_tables(int nrings, const int* __restrict__ rings, const int* __restrict__ fft_n,
                                   const int64_t* __restrict__ chirp_off,
                                   const int64_t* __restrict__ bhat_off, const double2* __restrict__ tw,
                                   double2* __restrict__ chirp, double2* __restrict__ bhat,
                                   double2* __restrict__ scratch, int natural_max) {
  extern __shared__ double2 xs_sm[];
  for (int ri = blockIdx.x; ri < nrings; ri += gridDim.x) {
  const int k = rings[ri];
  const int n = 2 * k + 1;
  const int N = fft_n[k];
  const int logN = 31 - __clz(N);
  double2* xs = scratch ? scratch + (size_t)blockIdx.x * N : xs_sm;
  double2* ch = chirp + chirp_off[k];
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int64_t r = ((int64_t)t * t) % (2 * (int64_t)n);
    double s, c;
    sincospi((double)r / (double)n, &s, &c);
    ch[t] = make_double2(c, s);
  }
  __syncthreads();
  for (int dir = 0; dir < 2; ++dir) {  // 0: forward analysis (b = chirp), 1: inverse (b = conj chirp)
    for (int u = threadIdx.x; u < N; u += blockDim.x) {
      int src = -1;
      if (u < n) src = u;
      else if (u > N - n) src = N - u;
      double2 b = make_double2(0.0, 0.0);
      if (src >= 0) {
        const int64_t r = ((int64_t)src * src) % (2 * (int64_t)n);
        double s, c;
        sincospi((double)r / (double)n, &s, &c);
        b = dir == 0 ? make_double2(c, s) : make_double2(c, -s);
      }
      xs[bitrev(u, logN)] = b;
    }
    fft_dit_smem(xs, N, logN, tw, false);
    const double inv = 1.0 / (double)N;
    double2* out = bhat + bhat_off[k] + (int64_t)dir * N;
    // bit-reversed order for the shared-memory transforms (bluestein_convolve), natural
    // order for the register-resident ones (N <= natural_max, fft_reg.cuh)
    // (N = 2048: even bins then odd bins, the two 1024-point halves of ringdft.cu's 2048 class)
    for (int u = threadIdx.x; u < N; u += blockDim.x) {
      int src = bitrev(u, logN);
      if (N <= natural_max) src = N == 2048 ? (u < 1024 ? 2 * u : 2 * (u - 1024) + 1) : u;
      const double2 v = xs[src];
      out[u] = make_double2(v.x * inv, v.y * inv);
    }
    __syncthreads();
  }
  }
}

static int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// OSPH_DEBUG_SYNC=1: synchronise after every table kernel and name the failing one
static cudaError_t dbg_sync(cudaStream_t st, const char* what) {
  static const bool on = getenv("OSPH_DEBUG_SYNC") != nullptr;
  if (!on) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) fprintf(stderr, "[osph] %s: %s\n", what, cudaGetErrorString(e));
  return e;
}

cudaError_t launch_tables(osph_plan* p) {
  const int L = p->L;
  cudaError_t e;
  cudaStream_t st = p->stream;
  if ((e = dbg_sync(st, "before tables")) != cudaSuccess) return e;
  {
    dim3 grid((L + 255) / 256, L);
    k_rec_table<<<grid, 256, 0, st>>>(L, p->d_rec);
    if ((e = dbg_sync(st, "k_rec_table")) != cudaSuccess) return e;
  }
  {
    double* seed_mant = nullptr;
    if ((e = cudaMallocAsync(&seed_mant, sizeof(double) * (size_t)L * L, st)) != cudaSuccess) return e;
    k_seeds<<<(L + 127) / 128, 128, 0, st>>>(L, p->d_sin, seed_mant, p->d_ls);
    if ((e = dbg_sync(st, "k_seeds")) != cudaSuccess) return e;
    dim3 grid((L + 127) / 128, L);
    k_start_table<<<grid, 128, 0, st>>>(L, p->d_cos, p->d_rec, seed_mant, p->d_ls, p->d_pstart);
    if ((e = dbg_sync(st, "k_start_table")) != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    cudaFreeAsync(seed_mant, st);
  }
  k_twiddles<<<(OSPH_TW_SIZE / 2 + 255) / 256, 256, 0, st>>>(p->d_tw);
  const int ndirect = std::min(L, (OSPH_DIRECT_MAX - 1) / 2 + 1);
  k_small_roots<<<ndirect, 64, 0, st>>>(ndirect, p->d_roots);
  if ((e = dbg_sync(st, "k_twiddles/k_small_roots")) != cudaSuccess) return e;
  k_stage_twiddles<<<OSPH_SW_GLOBAL / 2 / 256, 256, 0, st>>>(p->d_sw);
  k_reg_twiddles<<<(OSPH_RTW_SIZE + 255) / 256, 256, 0, st>>>(p->d_rtw);
  if ((e = dbg_sync(st, "k_stage_twiddles")) != cudaSuccess) return e;
  const int nsmall = p->n_bluestein_rings - p->n_big_rings;
  if (nsmall > 0) {
    int maxN = 0;
    for (int k = 0; k < L; ++k)
      if (p->h_fft_n[k] <= OSPH_FFT_MAX) maxN = std::max(maxN, p->h_fft_n[k]);
    const size_t smem = sizeof(double2) * (size_t)maxN;
    cudaFuncSetAttribute(k_bluestein_tables, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bluestein_tables<<<nsmall, 256, smem, st>>>(nsmall, p->d_bluestein_rings + p->n_big_rings, p->d_fft_n,
                                                  p->d_chirp_off, p->d_bhat_off, p->d_tw, p->d_chirp, p->d_bhat,
                                                  nullptr, p->reg_fft_max);
  }
  if (p->n_big_rings > 0) {  // 16384-point kernel spectra: work arrays in global memory
    const int nb = std::min(p->n_big_rings, 296);
    double2* scratch = nullptr;
    if ((e = cudaMallocAsync(&scratch, sizeof(double2) * (size_t)nb * 2 * OSPH_FFT_MAX, st)) != cudaSuccess)
      return e;
    k_bluestein_tables<<<nb, 256, 0, st>>>(p->n_big_rings, p->d_bluestein_rings, p->d_fft_n, p->d_chirp_off,
                                           p->d_bhat_off, p->d_tw, p->d_chirp, p->d_bhat, scratch, 0);
    cudaFreeAsync(scratch, st);
  }
  return cudaGetLastError();
}

// Host-side sizing of the ring-DFT tables (called by plan creation before upload).
void plan_dft_layout(osph_plan* p, std::vector<int>& bluestein_rings) {
  const int L = p->L;
  p->h_fft_n.assign(L, 0);
  p->h_chirp_off.assign(L, 0);
  p->h_bhat_off.assign(L, 0);
  int64_t coff = 0, boff = 0;
  bluestein_rings.clear();
  p->n_direct_rings = 0;
  for (int k = 0; k < L; ++k) {
    const int n = 2 * k + 1;
    if (n <= OSPH_DIRECT_MAX) {
      p->n_direct_rings++;
      continue;
    }
    const int N = next_pow2(2 * n - 1);
    p->h_fft_n[k] = N;
    p->h_chirp_off[k] = coff;
    p->h_bhat_off[k] = boff;
    coff += n;
    boff += 2 * (int64_t)N;
    bluestein_rings.push_back(k);
  }
  std::reverse(bluestein_rings.begin(), bluestein_rings.end());  // largest first
  p->n_bluestein_rings = (int)bluestein_rings.size();
  p->h_chirp_off.push_back(coff);
  p->h_bhat_off.push_back(boff);
}
