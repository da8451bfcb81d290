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
// Bluestein (chirp-z) with a power-of-two FFT in shared memory.
#include "fft.cuh"
#include "plan.cuh"

#define RING_THREADS 256

// Fold G (layout [m][k][4B]) of ring k, map b into bin t (t < n).
__device__ __forceinline__ double2 fold_bin(const double* __restrict__ G, int L, int B, int k, int n,
                                            int b, int t) {
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

// x (natural order) *= bhat, then permute to bit-reversed order in place.
__device__ __forceinline__ void mul_and_bitrev(double2* x, const double2* __restrict__ bh, int N, int logN) {
  for (int q = threadIdx.x; q < N; q += blockDim.x) x[q] = cmul(x[q], __ldg(bh + q));
  __syncthreads();
  for (int q = threadIdx.x; q < N; q += blockDim.x) {
    const int r = bitrev(q, logN);
    if (q < r) {
      const double2 a = x[q];
      x[q] = x[r];
      x[r] = a;
    }
  }
}

__global__ void __launch_bounds__(RING_THREADS) k_ring_inverse_bluestein(
    int L, int B, int maps_per_block, const int* __restrict__ rings, const int* __restrict__ fft_n,
    const int64_t* __restrict__ chirp_off, const int64_t* __restrict__ bhat_off,
    const double2* __restrict__ chirp_all, const double2* __restrict__ bhat_all,
    const double2* __restrict__ tw, const double* __restrict__ G, double2* __restrict__ samples) {
  extern __shared__ double2 xs[];
  const int k = rings[blockIdx.x];
  const int n = 2 * k + 1;
  const int N = fft_n[k];
  const int logN = 31 - __clz(N);
  const double2* chirp = chirp_all + chirp_off[k];
  const double2* bh = bhat_all + bhat_off[k] + N;  // inverse-direction kernel
  const int b0 = blockIdx.y * maps_per_block;
  const int b1 = min(B, b0 + maps_per_block);
  for (int b = b0; b < b1; ++b) {
    for (int t = threadIdx.x; t < N; t += blockDim.x) {
      double2 v = make_double2(0.0, 0.0);
      if (t < n) v = cmul(fold_bin(G, L, B, k, n, b, t), __ldg(chirp + t));
      xs[bitrev(t, logN)] = v;
    }
    fft_dit_smem(xs, N, logN, tw, false);
    mul_and_bitrev(xs, bh, N, logN);
    fft_dit_smem(xs, N, logN, tw, true);
    double2* out = samples + (int64_t)b * L * L + (int64_t)k * k;
    for (int j = threadIdx.x; j < n; j += blockDim.x) out[j] = cmul(xs[j], __ldg(chirp + j));
    __syncthreads();
  }
}

__global__ void __launch_bounds__(RING_THREADS) k_ring_inverse_direct(
    int L, int B, int nrings, int maps_per_block, const double2* __restrict__ roots,
    const double* __restrict__ G, double2* __restrict__ samples) {
  __shared__ double2 bins[OSPH_DIRECT_MAX + 1];
  const int k = blockIdx.x;
  const int n = 2 * k + 1;
  const int b0 = blockIdx.y * maps_per_block;
  const int b1 = min(B, b0 + maps_per_block);
  const double2* rt = roots + (int64_t)k * k;
  for (int b = b0; b < b1; ++b) {
    for (int t = threadIdx.x; t < n; t += blockDim.x) bins[t] = fold_bin(G, L, B, k, n, b, t);
    __syncthreads();
    double2* out = samples + (int64_t)b * L * L + (int64_t)k * k;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double re = 0.0, im = 0.0;
      int idx = 0;
      for (int t = 0; t < n; ++t) {  // e^{+2 pi i t j / n}
        const double2 w = rt[idx];
        const double2 v = bins[t];
        re += v.x * w.x - v.y * w.y;
        im += v.x * w.y + v.y * w.x;
        idx += j;
        if (idx >= n) idx -= n;
      }
      out[j] = make_double2(re, im);
    }
    __syncthreads();
  }
}

// Scatter one ring spectrum (forward sign, unnormalised) into the RHS layout.
__device__ __forceinline__ void scatter_rhs(const double2* X, int L, int B, int k, int n, int b,
                                            double2* __restrict__ R) {
  const double scale = OSPH_TWO_PI / (double)n;
  for (int m = threadIdx.x; m <= k; m += blockDim.x) {
    const double2 xp = X[m];
    const double2 xn = X[m == 0 ? 0 : n - m];
    const int64_t base = (packed_pos(L, m, k - m) * 2) * B + b;
    R[base] = make_double2(scale * xp.x, scale * xp.y);
    R[base + B] = make_double2(scale * xn.x, scale * xn.y);
  }
}

__global__ void __launch_bounds__(RING_THREADS) k_ring_forward_bluestein(
    int L, int B, int maps_per_block, const int* __restrict__ rings, const int* __restrict__ fft_n,
    const int64_t* __restrict__ chirp_off, const int64_t* __restrict__ bhat_off,
    const double2* __restrict__ chirp_all, const double2* __restrict__ bhat_all,
    const double2* __restrict__ tw, const double2* __restrict__ samples, double2* __restrict__ R) {
  extern __shared__ double2 xs[];
  const int k = rings[blockIdx.x];
  const int n = 2 * k + 1;
  const int N = fft_n[k];
  const int logN = 31 - __clz(N);
  const double2* chirp = chirp_all + chirp_off[k];
  const double2* bh = bhat_all + bhat_off[k];  // forward-direction kernel
  const int b0 = blockIdx.y * maps_per_block;
  const int b1 = min(B, b0 + maps_per_block);
  for (int b = b0; b < b1; ++b) {
    const double2* in = samples + (int64_t)b * L * L + (int64_t)k * k;
    for (int t = threadIdx.x; t < N; t += blockDim.x) {
      double2 v = make_double2(0.0, 0.0);
      if (t < n) v = cmul(__ldg(in + t), conj2(__ldg(chirp + t)));
      xs[bitrev(t, logN)] = v;
    }
    fft_dit_smem(xs, N, logN, tw, false);
    mul_and_bitrev(xs, bh, N, logN);
    fft_dit_smem(xs, N, logN, tw, true);
    for (int j = threadIdx.x; j < n; j += blockDim.x) xs[j] = cmul(xs[j], conj2(__ldg(chirp + j)));
    __syncthreads();
    scatter_rhs(xs, L, B, k, n, b, R);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(RING_THREADS) k_ring_forward_direct(
    int L, int B, int maps_per_block, const double2* __restrict__ roots, const double2* __restrict__ samples,
    double2* __restrict__ R) {
  __shared__ double2 xin[OSPH_DIRECT_MAX + 1];
  __shared__ double2 X[OSPH_DIRECT_MAX + 1];
  const int k = blockIdx.x;
  const int n = 2 * k + 1;
  const int b0 = blockIdx.y * maps_per_block;
  const int b1 = min(B, b0 + maps_per_block);
  const double2* rt = roots + (int64_t)k * k;
  for (int b = b0; b < b1; ++b) {
    const double2* in = samples + (int64_t)b * L * L + (int64_t)k * k;
    for (int t = threadIdx.x; t < n; t += blockDim.x) xin[t] = in[t];
    __syncthreads();
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      double re = 0.0, im = 0.0;
      int idx = 0;
      for (int t = 0; t < n; ++t) {  // e^{-2 pi i q t / n}
        const double2 w = rt[idx];
        const double2 v = xin[t];
        re += v.x * w.x + v.y * w.y;
        im += v.y * w.x - v.x * w.y;
        idx += q;
        if (idx >= n) idx -= n;
      }
      X[q] = make_double2(re, im);
    }
    __syncthreads();
    scatter_rhs(X, L, B, k, n, b, R);
    __syncthreads();
  }
}

static int max_fft(const osph_plan* p) {
  int N = 0;
  for (int v : p->h_fft_n) N = v > N ? v : N;
  return N;
}

static int maps_per_block_for(int B, int rings) {
  // keep >= ~4 waves of blocks on 148 SMs while amortising table reads
  int mpb = 1;
  while (mpb < 8 && (int64_t)rings * ((B + 2 * mpb - 1) / (2 * mpb)) >= 148 * 8) mpb *= 2;
  return mpb;
}

cudaError_t launch_ring_inverse(osph_plan* p, int B, double2* samples) {
  const int L = p->L;
  if (p->n_bluestein_rings > 0) {
    const int mpb = maps_per_block_for(B, p->n_bluestein_rings);
    const size_t smem = sizeof(double2) * (size_t)max_fft(p);
    cudaFuncSetAttribute(k_ring_inverse_bluestein, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(p->n_bluestein_rings, (B + mpb - 1) / mpb);
    k_ring_inverse_bluestein<<<grid, RING_THREADS, smem, p->stream>>>(
        L, B, mpb, p->d_bluestein_rings, p->d_fft_n, p->d_chirp_off, p->d_bhat_off, p->d_chirp, p->d_bhat,
        p->d_tw, p->d_g, samples);
    p->launches++;
  }
  if (p->n_direct_rings > 0) {
    const int mpb = maps_per_block_for(B, p->n_direct_rings);
    dim3 grid(p->n_direct_rings, (B + mpb - 1) / mpb);
    k_ring_inverse_direct<<<grid, 64, 0, p->stream>>>(L, B, p->n_direct_rings, mpb, p->d_roots, p->d_g,
                                                      samples);
    p->launches++;
  }
  return cudaGetLastError();
}

cudaError_t launch_ring_forward(osph_plan* p, int B, const double2* samples) {
  const int L = p->L;
  if (p->n_bluestein_rings > 0) {
    const int mpb = maps_per_block_for(B, p->n_bluestein_rings);
    const size_t smem = sizeof(double2) * (size_t)max_fft(p);
    cudaFuncSetAttribute(k_ring_forward_bluestein, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(p->n_bluestein_rings, (B + mpb - 1) / mpb);
    k_ring_forward_bluestein<<<grid, RING_THREADS, smem, p->stream>>>(
        L, B, mpb, p->d_bluestein_rings, p->d_fft_n, p->d_chirp_off, p->d_bhat_off, p->d_chirp, p->d_bhat,
        p->d_tw, samples, p->d_r);
    p->launches++;
  }
  if (p->n_direct_rings > 0) {
    const int mpb = maps_per_block_for(B, p->n_direct_rings);
    dim3 grid(p->n_direct_rings, (B + mpb - 1) / mpb);
    k_ring_forward_direct<<<grid, 64, 0, p->stream>>>(L, B, mpb, p->d_roots, samples, p->d_r);
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
