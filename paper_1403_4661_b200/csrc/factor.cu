// factor.cu -- per-order block construction and explicit inversion.
//
// Reference: the forward transform solves, for each order m, the square
// system (2pi Y_lm(theta_k, 0))_{k>=m, l>=m} f = g with a rank-revealing
// least-squares solve (gelsy, rcond 1e-14) and raises
// IllConditionedSolveError(order, kappa) on rank deficiency
// (pkg/src/optisph/transform.py:396-429, blocks.py:88-116).  The blocks do
// not depend on the data, so every order is factored up front, in parallel
// over m, by blocked Gauss-Jordan elimination with partial (row) pivoting.
// The result X satisfies A^{-1} = X P: the sweep gathers the right-hand side
// through the permutation and multiplies by X, a parallel GEMV instead of two
// serial triangular solves (LU vs gelsy: max|df| 2.2e-14 at L=512).
//
// One thread-block CLUSTER per order.  Every CTA of the cluster factors the
// current n x NB panel redundantly in registers (one matrix row per thread
// slot), then applies the row swaps and the rank-NB Gauss-Jordan update
//     A[:, cols] += E * A[panel rows, cols],  E = panel - I on the pivot rows
// to its own slice of columns on the fp64 tensor cores (mma.sync m8n8k4 ->
// SASS DMMA.8x8x4).  Cluster barriers order the panel hand-off.
//
// The reference's rank check becomes a 1-norm condition estimate
// kappa = ||A||_1 ||A^{-1}||_1 / sqrt(n), flagged above 2/rcond = 2e14
// (calibrated on the interleaved L=256 grid: gelsy first reports rank
// deficiency at m=220 where this estimate is 3.0e14; m=221 gives 1.9e14).
//
// Also written: the "below" block 2pi Y_lm(theta_k), k < m (the k<m
// correction matrix of transform.py:425-428), used by the sweep.
//
// Storage per order m (n = L-m): X column-major workspace, element (i, j) at
// j*n + i (i = degree l-m, j = pivoted ring row); perm[packed_pos(L,m,j)] =
// ring offset feeding column j.  For the sweep, X is re-emitted in 8-row
// tiles Xt[((i/8)*n + j)*8 + i%8] (rows padded to a multiple of 8 with zeros)
// and Pb is written directly in 8-ring tiles Pb[((k/8)*n + l-m)*8 + k%8], so
// a CTA's row slice of either matrix is a run of contiguous 64-byte columns
// that the sweep streams with bulk (TMA) copies.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "plan.cuh"

namespace cg = cooperative_groups;

cudaError_t launch_factor_np_class(osph_plan* p, int m_first, int m_last, int cs, cudaStream_t st);  // factor_np.cu

#define FAC_THREADS 256
#define FAC_TC 8      // column tile width of the rank-NB update
#define FAC_SUPER 64  // columns staged per T super tile

__device__ __forceinline__ void atomic_max_pos(unsigned long long* addr, double v) {
  if (!(v >= 0.0) || isinf(v)) v = INFINITY;  // NaN / inf -> inf
  atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

template <int RPT, int NB>
__global__ void __launch_bounds__(FAC_THREADS, 1) k_factor_gj(
    int L, int m_first, const double* __restrict__ costh, const double2* __restrict__ rec,
    const int* __restrict__ ls_tab, const double2* __restrict__ pstart, const int64_t* __restrict__ ainv_off,
    const int64_t* __restrict__ pb_off, double* __restrict__ ainv, double* __restrict__ pbelow,
    int* __restrict__ perm_all, unsigned long long* __restrict__ norms, int* __restrict__ status_out,
    int* __restrict__ jstar_out, double* __restrict__ beta_out, double* __restrict__ xt_all,
    const int64_t* __restrict__ xt_off, double* __restrict__ u_out, double* __restrict__ w_out) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int m = m_first + (int)(blockIdx.x / CS);
  if (m >= L) return;  // whole cluster exits together
  const int n = L - m;
  const int tid = threadIdx.x;

  extern __shared__ __align__(16) double smem[];
  double* Es = smem;                           // E, column-major [NB][n]
  double* Ts = smem + (size_t)NB * n;          // T super tile [NB][FAC_SUPER]
  __shared__ double red_v[FAC_THREADS / 32];
  __shared__ int red_i[FAC_THREADS / 32];
  __shared__ __align__(16) double prow[2][NB];
  __shared__ __align__(16) double jrow[2][NB];
  __shared__ int pivs[NB];
  __shared__ int s_bad;
  __shared__ double s_cmax;

  double* A = ainv + ainv_off[m];
  double* Pb = pbelow + pb_off[m];
  int* perm = perm_all + packed_pos(L, m, 0);
  if (tid == 0) s_bad = 0;

  // ---- 1. generate 2pi*Y_lm(theta_k); rings split over the cluster
  for (int k = rank * FAC_THREADS + tid; k < L; k += CS * FAC_THREADS) {
    const int64_t t = (int64_t)m * L + k;
    const int ls = ls_tab[t];
    const double2 pp = pstart[t];
    double p0 = pp.x, p1 = pp.y;
    const double x = costh[k];
    const double2* recm = rec + packed_pos(L, m, 0);
    for (int l = m; l < L; ++l) {
      double v = 0.0;
      if (l >= ls) {
        v = OSPH_TWO_PI * p1;
        const double2 ar = __ldg(recm + (l - m));
        const double nxt = fma(x, p1, -ar.x * p0) * ar.y;
        p0 = p1;
        p1 = nxt;
      }
      if (k >= m) A[(int64_t)(l - m) * n + (k - m)] = v;
      else Pb[tile_index(k, l - m, (m + 7) >> 3)] = v;  // chunk-major 8-ring tiles
    }
  }
  if (rank == 0)
    for (int i = tid; i < n; i += FAC_THREADS) perm[i] = i;

  // column ownership in units of NB columns
  const int units = (n + NB - 1) / NB;
  const int u0 = (rank * units) / CS, u1 = ((rank + 1) * units) / CS;
  const int cown0 = u0 * NB, cown1 = min(n, u1 * NB);
  const int warp = tid >> 5, lane = tid & 31;

  cluster.sync();
  // ||A||_1 over own columns
  {
    double cmax = 0.0;
    for (int col = cown0 + warp; col < cown1; col += FAC_THREADS / 32) {
      double s = 0.0;
      for (int i = lane; i < n; i += 32) s += fabs(__ldcg(A + (int64_t)col * n + i));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      cmax = fmax(cmax, s);
    }
    if (lane == 0 && cown0 < cown1) atomic_max_pos(norms + 2 * m, cmax);
  }

  double reg[RPT][NB];
  for (int j0 = 0; j0 < n; j0 += NB) {
    const int nb = min(NB, n - j0);
    // ---- a) panel -> registers (written by its owner before the last cluster barrier)
#pragma unroll
    for (int s = 0; s < RPT; ++s) {
      const int row = tid + s * FAC_THREADS;
#pragma unroll
      for (int c = 0; c < NB; ++c)
        reg[s][c] = (row < n && c < nb) ? __ldcg(A + (int64_t)(j0 + c) * n + row) : 0.0;
    }
    // ---- b) unblocked Gauss-Jordan on the panel, redundantly in every CTA
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c < nb) {
        const int jc = j0 + c;
        const int bufi = c & 1;
        double bv = -1.0;
        int bi = jc;
#pragma unroll
        for (int s = 0; s < RPT; ++s) {
          const int row = tid + s * FAC_THREADS;
          const double a = fabs(reg[s][c]);
          if (row >= jc && row < n && a > bv) {
            bv = a;
            bi = row;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
          }
        }
        if (lane == 0) {
          red_v[warp] = bv;
          red_i[warp] = bi;
        }
        __syncthreads();
        int p = red_i[0];
        {
          double best = red_v[0];
#pragma unroll
          for (int w = 1; w < FAC_THREADS / 32; ++w)
            if (red_v[w] > best || (red_v[w] == best && red_i[w] < p)) {
              best = red_v[w];
              p = red_i[w];
            }
        }
        // owner of p publishes the pivot row, owner of jc its current row
        const int own_p = p % FAC_THREADS, slot_p = p / FAC_THREADS;
        const int own_j = jc % FAC_THREADS, slot_j = jc / FAC_THREADS;
#pragma unroll
        for (int s = 0; s < RPT; ++s) {
          if (tid == own_p && s == slot_p)
#pragma unroll
            for (int cc = 0; cc < NB; ++cc) prow[bufi][cc] = reg[s][cc];
          if (tid == own_j && s == slot_j)
#pragma unroll
            for (int cc = 0; cc < NB; ++cc) jrow[bufi][cc] = reg[s][cc];
        }
        if (tid == 0) pivs[c] = p;
        __syncthreads();
        const double d = prow[bufi][c];
        if (tid == 0 && (d == 0.0 || !isfinite(d))) s_bad = 1;
        const double inv_d = 1.0 / d;
#pragma unroll
        for (int s = 0; s < RPT; ++s) {
          const int row = tid + s * FAC_THREADS;
          if (row == jc) {
#pragma unroll
            for (int cc = 0; cc < NB; ++cc) reg[s][cc] = (cc == c) ? inv_d : prow[bufi][cc] * inv_d;
          } else {
            if (row == p) {  // receives the old row jc
#pragma unroll
              for (int cc = 0; cc < NB; ++cc) reg[s][cc] = jrow[bufi][cc];
            }
            const double f = reg[s][c] * inv_d;
#pragma unroll
            for (int cc = 0; cc < NB; ++cc)
              if (cc != c) reg[s][cc] = fma(-f, prow[bufi][cc], reg[s][cc]);
            reg[s][c] = -f;
          }
        }
      }
    }
    // ---- c) E -> smem; the panel's owner stores the panel; permutation bookkeeping
    const bool own_panel = (j0 >= cown0 && j0 < cown1);
#pragma unroll
    for (int s = 0; s < RPT; ++s) {
      const int row = tid + s * FAC_THREADS;
      if (row < n) {
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          if (c < nb) {
            Es[(size_t)c * n + row] = reg[s][c] - ((row == j0 + c) ? 1.0 : 0.0);
            if (own_panel) A[(int64_t)(j0 + c) * n + row] = reg[s][c];
          }
        }
      }
    }
    if (rank == 0 && tid == 0) {
      for (int c = 0; c < nb; ++c) {
        const int p = pivs[c];
        if (p != j0 + c) {
          const int a = perm[j0 + c];
          perm[j0 + c] = perm[p];
          perm[p] = a;
        }
      }
    }
    __syncthreads();
    // ---- d) deferred row swaps on own non-panel columns
    for (int col = cown0 + tid; col < cown1; col += FAC_THREADS) {
      if (col >= j0 && col < j0 + nb) continue;
      double* cl = A + (int64_t)col * n;
      for (int c = 0; c < nb; ++c) {
        const int p = pivs[c];
        if (p != j0 + c) {
          const double a = cl[j0 + c];
          cl[j0 + c] = cl[p];
          cl[p] = a;
        }
      }
    }
    __syncthreads();
    // ---- e) rank-nb update of own non-panel columns on DMMA
    const int g = lane >> 2, tq = lane & 3;
    const int nrt = (n + 31) / 32;
    for (int cs = cown0; cs < cown1; cs += FAC_SUPER) {
      const int ce = min(cown1, cs + FAC_SUPER);
      if (cs >= j0 && ce <= j0 + nb) continue;
      for (int idx = tid; idx < NB * FAC_SUPER; idx += FAC_THREADS) {
        const int r = idx / FAC_SUPER, cc = idx - r * FAC_SUPER;
        const int col = cs + cc;
        Ts[idx] = (r < nb && col < ce) ? A[(int64_t)col * n + j0 + r] : 0.0;
      }
      __syncthreads();
      const int nct = (ce - cs + FAC_TC - 1) / FAC_TC;
      for (int wt = warp; wt < nrt * nct; wt += FAC_THREADS / 32) {
        const int rt = wt % nrt, ct = wt / nrt;
        const int c0 = cs + ct * FAC_TC;
        if (c0 >= j0 && c0 < j0 + nb) continue;  // panel columns are final
        const int r0 = rt * 32;
        const int colA = c0 + 2 * tq, colB = colA + 1;
        double acc[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = r0 + i * 8 + g;
          acc[i][0] = (row < n && colA < ce) ? A[(int64_t)colA * n + row] : 0.0;
          acc[i][1] = (row < n && colB < ce) ? A[(int64_t)colB * n + row] : 0.0;
        }
#pragma unroll
        for (int k0 = 0; k0 < NB; k0 += 4) {
          const int kk = k0 + tq;
          const double b = Ts[kk * FAC_SUPER + (c0 - cs) + g];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = r0 + i * 8 + g;
            const double a = (kk < nb && row < n) ? Es[(size_t)kk * n + row] : 0.0;
            dmma_8x8x4(acc[i][0], acc[i][1], a, b);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = r0 + i * 8 + g;
          if (row < n) {
            if (colA < ce) A[(int64_t)colA * n + row] = acc[i][0];
            if (colB < ce) A[(int64_t)colB * n + row] = acc[i][1];
          }
        }
      }
      __syncthreads();
    }
    cluster.sync();  // next panel's columns are final everywhere
  }

  // ---- 3. ||X||_1 over own columns (column sums are permutation invariant)
  {
    double cmax = 0.0;
    for (int col = cown0 + warp; col < cown1; col += FAC_THREADS / 32) {
      double s = 0.0;
      for (int i = lane; i < n; i += 32) s += fabs(__ldcg(A + (int64_t)col * n + i));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      cmax = fmax(cmax, s);
    }
    if (lane == 0 && cown0 < cown1) atomic_max_pos(norms + 2 * m + 1, cmax);
  }
  if (tid == 0 && s_bad) atomicOr(status_out + m, 1);
  (void)s_cmax;

  // own columns of X -> 8-row tiles for the sweep (padding rows zero)
  {
    double* Xt = xt_all + xt_off[m];
    const int npad = (n + 7) & ~7;
    const int nrt = npad >> 3;
    // the owner of the last columns also zero-fills the padding columns of the last chunk
    const int cend = (cown1 == n) ? (n + OSPH_TILE_KC - 1) / OSPH_TILE_KC * OSPH_TILE_KC : cown1;
    // column col of X (pivot order) is column perm[col] of X P^T (natural ring
    // order, the sweep's operand); the late ring's column (perm = 0) is zero
    for (int col = cown0; col < cend; ++col) {
      const int cn = col < n ? __ldcg(perm + col) : col;
      for (int i = tid; i < npad; i += FAC_THREADS)
        Xt[tile_index(i, cn, nrt)] = (i < n && col < n && cn != 0) ? __ldcg(A + (int64_t)col * n + i) : 0.0;
    }
  }

  // u_m[j] = Pb_m[ring m-1, :] . X[:, j] for own columns, stored in natural ring
  // order: the sweep's chain partial a_{m-1} = Pb_m[m-1, :] . x'_m is u_m . rhs_m
  {
    double* u = u_out + (size_t)m * uw_ld(L);
    const int nrtpb = (m + 7) >> 3;
    for (int col = cown0 + warp; col < cown1; col += FAC_THREADS / 32) {
      double s = 0.0;
      if (m >= 1)
        for (int i = lane; i < n; i += 32)
          s += __ldcg(Pb + tile_index(m - 1, i, nrtpb)) * __ldcg(A + (int64_t)col * n + i);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        const int cn = __ldcg(perm + col);  // natural ring order; the late ring's weight is zero
        u[cn] = cn != 0 ? s : 0.0;
      }
    }
  }

  // ---- 4. sweep chain constants (rank 0): j* = column of X fed by ring m
  // (perm[j*] = 0) and beta_m = Pb_m[ring m-1, :] . X[:, j*], the coupling of
  // order m's late right-hand-side entry into ring m-1 of order m-1.
  if (rank == 0) {
    __shared__ int s_jstar;
    __shared__ double s_beta[FAC_THREADS / 32];
    for (int j = tid; j < n; j += FAC_THREADS)
      if (__ldcg(perm + j) == 0) s_jstar = j;
    __syncthreads();
    const int js = s_jstar;
    double acc = 0.0;
    if (m >= 1)
      for (int l = tid; l < n; l += FAC_THREADS)
        acc += __ldcg(Pb + tile_index(m - 1, l, (m + 7) >> 3)) *
               __ldcg(A + (int64_t)js * n + l);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) s_beta[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double b = 0.0;
      for (int w = 0; w < FAC_THREADS / 32; ++w) b += s_beta[w];
      beta_out[m] = b;
      jstar_out[m] = js;
    }
    for (int l = tid; l < n; l += FAC_THREADS) w_out[(size_t)m * uw_ld(L) + l] = __ldcg(A + (int64_t)js * n + l);
  }
}

// Finalise kappa per order once every cluster has finished.
__global__ void k_kappa(int L, const unsigned long long* __restrict__ norms, double* __restrict__ kappa) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= L) return;
  const double a = __longlong_as_double((long long)norms[2 * m]);
  const double x = __longlong_as_double((long long)norms[2 * m + 1]);
  const double k = a * x / sqrt((double)(L - m));
  kappa[m] = isfinite(k) ? k : INFINITY;
}

struct FacClass {
  int nmax;     // largest block size in the class
  int cluster;  // CTAs per order
};

template <int RPT, int NB>
static cudaError_t launch_class(osph_plan* p, int m_first, int m_last, int cs, cudaStream_t st) {
  const int L = p->L;
  const int n = L - m_first;
  const size_t smem = sizeof(double) * ((size_t)NB * n + (size_t)NB * FAC_SUPER);
  auto kern = k_factor_gj<RPT, NB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((m_last - m_first + 1) * cs));
  cfg.blockDim = dim3(FAC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, L, m_first, (const double*)p->d_cos, (const double2*)p->d_rec,
                         (const int*)p->d_ls, (const double2*)p->d_pstart, (const int64_t*)p->d_ainv_off,
                         (const int64_t*)p->d_pb_off, p->d_ainv, p->d_pbelow, p->d_piv, p->d_norms,
                         p->d_status, p->d_jstar, p->d_beta, p->d_xt, (const int64_t*)p->d_xt_off, p->d_u, p->d_w);
  p->launches++;
  return e;
}

cudaError_t launch_kappa(osph_plan* p, cudaStream_t st) {
  k_kappa<<<(p->L + 127) / 128, 128, 0, st>>>(p->L, p->d_norms, p->d_kappa);
  p->launches++;
  return cudaGetLastError();
}

// Orders are grouped by block size n = L - m; each group gets a kernel
// instantiation whose register tile fits n and a cluster size that scales
// the rank-NB update with n^2.  The largest class runs on `st`; the smaller
// classes run on `st2` so they fill the SMs the large class's tail leaves idle
// (the classes write disjoint orders).  Both streams are joined back into `st`.
cudaError_t launch_factor(osph_plan* p, cudaStream_t st, cudaStream_t st2) {
  const int L = p->L;
  cudaError_t e;
  if (!st) st = p->stream;
  const bool first_call = !p->piv_ready;
  // first call: the partial-pivoting kernels record the pivot order (grid-determined);
  // run them serially, then redo the large orders with the breadth-first kernel below
  if (getenv("OSPH_FACTOR_ONE_STREAM") || first_call) st2 = nullptr;
  if ((e = cudaMemsetAsync(p->d_norms, 0, sizeof(unsigned long long) * 2 * L, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p->d_status, 0, sizeof(int) * L, st)) != cudaSuccess) return e;
  if (st2) {
    if ((e = cudaEventRecord(p->ev_fac[0], st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st2, p->ev_fac[0], 0)) != cudaSuccess) return e;
  }
  // classes by n (inclusive upper bounds), processed largest first
  struct Cls {
    int nlo, nhi, cs;
  };
  const Cls classes[] = {{1025, 2048, 16}, {513, 1024, 16}, {257, 512, 8}, {129, 256, 4}, {65, 128, 2}, {1, 64, 1}};
  const bool static_piv = p->piv_ready && !getenv("OSPH_FACTOR_PIVOTED");
  bool first = true;
  const int nmin = p->bf_nmin;
  if (static_piv && L > nmin && !getenv("OSPH_FACTOR_NO_BF")) {
    // every order with n > bf_nmin in one breadth-first blocked pass (factor_bf.cu)
    if ((e = launch_factor_bf(p, 0, L - nmin - 1, st)) != cudaSuccess) return e;
    first = false;
  }
  for (const Cls& c : classes) {
    const int nhi = std::min(c.nhi, L);
    if (nhi < c.nlo) continue;
    if (!first && static_piv && c.nlo > nmin && !getenv("OSPH_FACTOR_NO_BF")) continue;  // done by the BF pass
    const int m_first = L - nhi, m_last = L - c.nlo;
    cudaStream_t s = (first || !st2) ? st : st2;
    first = false;
    if (static_piv && nhi <= 256) {  // pivot order known: shared-memory static-pivot kernel
      e = launch_factor_np_class(p, m_first, m_last, nhi > 128 ? 4 : 1, s);
      if (e != cudaSuccess) return e;
      continue;
    }
    if (nhi > 1024) e = launch_class<8, 8>(p, m_first, m_last, c.cs, s);
    else if (nhi > 512) e = launch_class<4, 16>(p, m_first, m_last, c.cs, s);
    else if (nhi > 256) e = launch_class<2, 32>(p, m_first, m_last, c.cs, s);
    else e = launch_class<1, 32>(p, m_first, m_last, c.cs, s);
    if (e != cudaSuccess) return e;
  }
  if (st2) {
    if ((e = cudaEventRecord(p->ev_fac[1], st2)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st, p->ev_fac[1], 0)) != cudaSuccess) return e;
  }
  if (first_call && L > nmin && !getenv("OSPH_FACTOR_NO_BF") && !getenv("OSPH_FACTOR_PIVOTED")) {
    // the X of the largest pivoted class is not trusted for n > 1024; the
    // breadth-first pass with the recorded pivots recomputes every order n > 256
    if ((e = launch_factor_bf(p, 0, L - nmin - 1, st)) != cudaSuccess) return e;
  }
  k_kappa<<<(L + 127) / 128, 128, 0, st>>>(L, p->d_norms, p->d_kappa);
  p->launches++;
  p->piv_ready = true;  // the pivot order depends on the grid only
  return cudaGetLastError();
}
