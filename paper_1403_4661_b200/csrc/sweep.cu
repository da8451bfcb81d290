// sweep.cu -- the order-peeling sweep of the forward transform.
//
// Reference: _forward_spectral (pkg/src/optisph/transform.py:436-467), with
// the solve of _solve_pair/solve_columns (transform.py:396-406,
// blocks.py:94-116).  For m = L-1 .. 0:
//   g_(+-m)[k-m] = (2pi/n_k) X_k[+-m mod n_k], k >= m      (445-449)
//   [f_m, f_-m] = A_m^{-1} [g_+m, (-1)^m g_-m]              (451)
//   G_(+-m)(theta_k) = 2pi sum_l Y_lm(theta_k) f_l(+-m), k < m  (455-458)
//   X_k[+-m mod n_k] -= n_k G_(+-m)/2pi                     (459-463)
// The ring spectra are held in the order-major RHS layout R (ringdft.cu), in
// which the bin update is simply R[target] -= G and the RHS of order m is the
// contiguous slab R[pos(m, 0..n)].
//
// A "team" (one thread-block cluster) owns a group of maps and runs the whole
// sweep with cluster barriers only; teams are independent, so a batch fills
// the GPU with teams (maps) and a single map gets one 16-CTA team.  Per order:
//   phase 1: x = X * (P rhs)   rows of X split over the team   (solve)
//   phase 2: G = Pb * x        rings k < m split over the team (correction)
#include <cooperative_groups.h>

#include <algorithm>

#include "plan.cuh"

namespace cg = cooperative_groups;

#define SWEEP_THREADS 256

template <int CC>
__global__ void __launch_bounds__(SWEEP_THREADS) k_sweep(
    int L, int B, int maps_per_team, const double* __restrict__ ainv, const int64_t* __restrict__ ainv_off,
    const int* __restrict__ perm_all, const double* __restrict__ pbelow, const int64_t* __restrict__ pb_off,
    double2* __restrict__ R, double* __restrict__ xs_all, double2* __restrict__ flm) {
  cg::cluster_group cluster = cg::this_cluster();
  const int T = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int team = (int)(blockIdx.x / T);
  const int b0 = team * maps_per_team;
  const int gm = min(maps_per_team, B - b0);
  const int tid = threadIdx.x;
  extern __shared__ __align__(16) double vec[];  // [L][CC]: rhs in phase 1, x in phase 2
  double* xg = xs_all + (int64_t)team * L * CC;

  for (int m = L - 1; m >= 0; --m) {
    const int n = L - m;
    const double sgn = (m & 1) ? -1.0 : 1.0;
    const int64_t pm = packed_pos(L, m, 0);
    const int* perm = perm_all + pm;
    // ---- phase 1: permuted right-hand side -> smem
    for (int idx = tid; idx < n * (CC / 4); idx += SWEEP_THREADS) {
      const int i = idx / (CC / 4), bl = idx - i * (CC / 4);
      double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
      if (bl < gm) {
        const int64_t base = ((pm + perm[i]) * 2) * B + b0 + bl;
        const double2 rp = __ldcg(R + base);
        const double2 rn = __ldcg(R + base + B);
        v = make_double4(rp.x, rp.y, sgn * rn.x, sgn * rn.y);
      }
      *reinterpret_cast<double4*>(vec + (size_t)i * CC + 4 * bl) = v;
    }
    __syncthreads();
    const double* X = ainv + ainv_off[m];
    const int r0 = (rank * n) / T, r1 = ((rank + 1) * n) / T;
    for (int l = r0 + tid; l < r1; l += SWEEP_THREADS) {
      double acc[CC];
#pragma unroll
      for (int c = 0; c < CC; ++c) acc[c] = 0.0;
      const double* xc = X + l;
      for (int i = 0; i < n; ++i) {
        const double a = __ldg(xc + (int64_t)i * n);
        const double* rv = vec + (size_t)i * CC;
#pragma unroll
        for (int c = 0; c < CC; ++c) acc[c] = fma(a, rv[c], acc[c]);
      }
#pragma unroll
      for (int c = 0; c < CC; ++c) xg[(size_t)l * CC + c] = acc[c];
      const int64_t ell = m + l;
      for (int bl = 0; bl < gm; ++bl) {
        double2* f = flm + (int64_t)(b0 + bl) * L * L + ell * ell + ell;
        f[m] = make_double2(acc[4 * bl], acc[4 * bl + 1]);
        if (m > 0) f[-m] = make_double2(acc[4 * bl + 2], acc[4 * bl + 3]);
      }
    }
    cluster.sync();
    if (m == 0) break;
    // ---- phase 2: corrections for rings k < m
    for (int idx = tid; idx < n * CC; idx += SWEEP_THREADS) vec[idx] = __ldcg(xg + idx);
    __syncthreads();
    const double* Pb = pbelow + pb_off[m];
    const int k0 = (rank * m) / T, k1 = ((rank + 1) * m) / T;
    for (int k = k0 + tid; k < k1; k += SWEEP_THREADS) {
      double acc[CC];
#pragma unroll
      for (int c = 0; c < CC; ++c) acc[c] = 0.0;
      for (int l = 0; l < n; ++l) {
        const double a = __ldg(Pb + (int64_t)l * m + k);
        const double* xv = vec + (size_t)l * CC;
#pragma unroll
        for (int c = 0; c < CC; ++c) acc[c] = fma(a, xv[c], acc[c]);
      }
      const int nk = 2 * k + 1;
      const int r = m % nk;
      int tm, tp_slot, tn_slot;  // target order; R slot receiving G+ and G-
      if (r == 0) {
        tm = 0;
        tp_slot = 0;
        tn_slot = 0;
      } else if (r <= k) {
        tm = r;
        tp_slot = 0;
        tn_slot = 1;
      } else {
        tm = nk - r;
        tp_slot = 1;
        tn_slot = 0;
      }
      const int64_t tbase = packed_pos(L, tm, k - tm) * 2 * B + b0;
      for (int bl = 0; bl < gm; ++bl) {
        const double2 gp = make_double2(acc[4 * bl], acc[4 * bl + 1]);
        const double2 gn = make_double2(sgn * acc[4 * bl + 2], sgn * acc[4 * bl + 3]);
        double2* rp = R + tbase + tp_slot * B + bl;
        double2 v = __ldcg(rp);
        v.x -= gp.x;
        v.y -= gp.y;
        if (tn_slot == tp_slot) {
          v.x -= gn.x;
          v.y -= gn.y;
          *rp = v;
        } else {
          *rp = v;
          double2* rn = R + tbase + tn_slot * B + bl;
          double2 w = __ldcg(rn);
          w.x -= gn.x;
          w.y -= gn.y;
          *rn = w;
        }
      }
    }
    cluster.sync();
  }
}

template <int CC>
static cudaError_t launch_sweep_cc(osph_plan* p, int B, int g, int T, double2* flm) {
  const int L = p->L;
  const int teams = (B + g - 1) / g;
  const size_t smem = sizeof(double) * (size_t)L * CC;
  auto kern = k_sweep<CC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (T > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(teams * T));
  cfg.blockDim = dim3(SWEEP_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = p->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = T;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, L, B, g, (const double*)p->d_ainv, (const int64_t*)p->d_ainv_off,
                         (const int*)p->d_piv, (const double*)p->d_pbelow, (const int64_t*)p->d_pb_off, p->d_r,
                         p->d_x, flm);
  p->launches++;
  return e;
}

cudaError_t launch_sweep(osph_plan* p, int B, double2* flm) {
  const int g = B >= 4 ? 4 : B;
  const int teams = (B + g - 1) / g;
  int T = 1;
  while (T < 16 && teams * T * 2 <= 148 && T * 32 < p->L) T *= 2;
  if (g == 4 || B == 3) return launch_sweep_cc<16>(p, B, 4, T, flm);
  if (g == 2) return launch_sweep_cc<8>(p, B, 2, T, flm);
  return launch_sweep_cc<4>(p, B, 1, T, flm);
}
