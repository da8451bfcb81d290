// factor_bf.cu -- batched, breadth-first blocked Gauss-Jordan inversion of the
// large per-order blocks (n = L - m > 256) with the grid-determined pivot order.
//
// Same result as factor.cu / factor_np.cu (explicit X = (P A_m)^{-1}, A_m =
// 2pi Y_lm(theta_k), k >= m, l >= m; transform.py:416-429, blocks.py:88-116),
// organised for throughput instead of per-order latency.  With the pivot
// order known (recorded by the partial-pivoting kernel on the plan's first
// call; it depends only on the grid), row i of the working matrix is ring
// m + perm[i] and Gauss-Jordan needs no interchanges, so a panel step on the
// column block J = [j0, j0 + nb) is purely block-algebraic:
//     D = A[J, J]^{-1}                 (nb x nb, one CTA per order)
//     E = -A[:, J] D,  E[J] = D - I    (n x nb, parallel over row tiles)
//     A[:, K] += E A[J, K]   (K != J)  (rank-nb update, DMMA tiles)
//     A[:, J]  = E + I_J
// and every order with n > j0 takes the step in the same three launches.
// The update (2 n^2 nb flops per order and step, nb = 64) is the bulk of the
// work: 64 x 64 output tiles on the fp64 tensor cores (mma.sync m8n8k4 ->
// DMMA.8x8x4), operands staged in shared memory.  After the last step the
// epilogue emits the sweep operands exactly as factor_np.cu does (X in
// chunk-major 8-row tiles with natural-order columns, w_m, u_m, j*, beta_m)
// plus ||X||_1 for the condition estimate.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "plan.cuh"

#define BF_NB 64       // panel width
#define BF_T 64        // output tile (rows and columns)
#define BF_THREADS 256
#define BF_LDS (BF_NB + 4)  // padded smem row stride (doubles)

__device__ __forceinline__ void bf_atomic_max_pos(unsigned long long* addr, double v) {
  if (!(v >= 0.0) || isinf(v)) v = INFINITY;
  atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ uint32_t bf_smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bf_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(bf_smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void bf_cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// E panels keep an even column stride so 16-byte async copies stay aligned.
__host__ __device__ __forceinline__ int bf_lde(int n) { return (n + 1) & ~1; }

// Work item lookup: order index within the launch from a prefix table of
// per-order item counts (binary search; pre[0] = 0, pre[cnt] = total).
// Warp-cooperative variant (a full warp calls it): 32-ary search, <= 3 rounds
// of one load per lane instead of ~11 dependent loads in one thread.
__device__ __forceinline__ int bf_find_warp(const int* __restrict__ pre, int cnt, int item) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = cnt;  // pre[lo] <= item < pre[hi]
  while (hi - lo > 1) {
    const int stride = (hi - lo + 31) >> 5;
    const int idx = lo + lane * stride;
    const bool ok = idx < hi && __ldg(pre + idx) <= item;
    const unsigned mask = __ballot_sync(0xffffffffu, ok);  // lane 0 (idx = lo) is always set
    lo += (31 - __clz(mask)) * stride;
    hi = min(hi, lo + stride);
  }
  return lo;
}

__device__ __forceinline__ int bf_find(const int* __restrict__ pre, int cnt, int item) {
  int lo = 0, hi = cnt;  // pre[lo] <= item < pre[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(pre + mid) <= item) lo = mid;
    else hi = mid;
  }
  return lo;
}

// ---- 1. the blocks: 2pi Y_lm(theta_{m + perm[i]}) at row i (column-major,
// column = degree l - m); rings k < m go to the tiled below-block Pb_m.
__global__ void __launch_bounds__(BF_THREADS) k_bf_generate(int L, int m_first, const double* __restrict__ costh,
                                                            const double2* __restrict__ rec,
                                                            const int* __restrict__ ls_tab,
                                                            const double2* __restrict__ pstart,
                                                            const int* __restrict__ perm_all,
                                                            const int64_t* __restrict__ ainv_off,
                                                            const int64_t* __restrict__ pb_off,
                                                            double* __restrict__ ainv, double* __restrict__ pbelow) {
  __shared__ double2 s_rec[BF_THREADS];  // recurrence factors of the current degree chunk (broadcast reads)
  const int m = m_first + blockIdx.y;
  const int n = L - m;
  const int t = blockIdx.x * BF_THREADS + threadIdx.x;
  const bool active = t < L;
  int k = 0, row = -1;
  if (active) {
    if (t < n) {
      row = t;
      k = m + __ldg(perm_all + packed_pos(L, m, t));
    } else {
      k = t - n;  // ring below the block
    }
  }
  double* A = ainv + __ldg(ainv_off + m);
  double* Pb = pbelow + __ldg(pb_off + m);
  const int64_t ts = (int64_t)m * L + k;
  const int ls = active ? __ldg(ls_tab + ts) : L;
  const double2 pp = active ? __ldg(pstart + ts) : make_double2(0.0, 0.0);
  double p0 = pp.x, p1 = pp.y;
  const double x = active ? __ldg(costh + k) : 0.0;
  const double2* recm = rec + packed_pos(L, m, 0);
  const int nrtpb = (m + 7) >> 3;
  for (int l0 = m; l0 < L; l0 += BF_THREADS) {
    __syncthreads();
    if (l0 + threadIdx.x < L) s_rec[threadIdx.x] = __ldg(recm + (l0 + threadIdx.x - m));
    __syncthreads();
    if (!active) continue;
    const int l1 = min(L, l0 + BF_THREADS);
    for (int l = l0; l < l1; ++l) {
      double v = 0.0;
      if (l >= ls) {
        v = OSPH_TWO_PI * p1;
        const double2 ar = s_rec[l - l0];
        const double nxt = fma(x, p1, -ar.x * p0) * ar.y;
        p0 = p1;
        p1 = nxt;
      }
      if (row >= 0) A[(int64_t)(l - m) * n + row] = v;
      else Pb[tile_index(k, l - m, nrtpb)] = v;
    }
  }
}

// A_m in natural ring order as chunk-major 8-ring tiles (the layout of X),
// for the large-L sweep's iterative refinement: thread = ring offset j.
__global__ void __launch_bounds__(BF_THREADS) k_bf_generate_at(int L, int m_first, const double* __restrict__ costh,
                                                               const double2* __restrict__ rec,
                                                               const int* __restrict__ ls_tab,
                                                               const double2* __restrict__ pstart,
                                                               const int64_t* __restrict__ at_off,
                                                               double* __restrict__ at) {
  const int m = m_first + blockIdx.y;
  const int n = L - m;
  const int j = blockIdx.x * BF_THREADS + threadIdx.x;
  if (j >= n) return;
  const int k = m + j;
  double* At = at + __ldg(at_off + m);
  const int nrt = (n + 7) >> 3;
  const int64_t ts = (int64_t)m * L + k;
  const int ls = __ldg(ls_tab + ts);
  const double2 pp = __ldg(pstart + ts);
  double p0 = pp.x, p1 = pp.y;
  const double x = __ldg(costh + k);
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
    At[tile_index(j, l - m, nrt)] = v;
  }
}

// ||A||_1 (or ||X||_1 after the sweep of panels): one warp per column.
__global__ void __launch_bounds__(BF_THREADS) k_bf_colnorm(int L, int m_first, const int64_t* __restrict__ ainv_off,
                                                           const double* __restrict__ ainv,
                                                           unsigned long long* __restrict__ norms, int which) {
  const int m = m_first + blockIdx.y;
  const int n = L - m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* A = ainv + __ldg(ainv_off + m);
  double cmax = 0.0;
  for (int c = blockIdx.x * (BF_THREADS / 32) + warp; c < n; c += gridDim.x * (BF_THREADS / 32)) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += fabs(__ldcg(A + (int64_t)c * n + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    cmax = fmax(cmax, s);
  }
  if (lane == 0 && cmax > 0.0) bf_atomic_max_pos(norms + 2 * m + which, cmax);
}

// ---- 2a. D = A[J, J]^{-1} (in-place Gauss-Jordan, no interchanges) and the
// row block R = A[J, :] (the update's B operand, snapshotted before the update).
// Grid (orders, column chunks of BF_RCHUNK): every block copies its chunk of R,
// block y = 0 also inverts D.  The inversion keeps a 4 x 4 patch of D per
// thread in registers; per pivot only the pivot row and column go through
// shared memory (double-buffered: one barrier per pivot).
#define BF_RCHUNK 256
__global__ void __launch_bounds__(BF_THREADS) k_bf_diag(int L, int m_first, int j0, const int64_t* __restrict__ ainv_off,
                                                        const double* __restrict__ ainv, double* __restrict__ dbuf,
                                                        double* __restrict__ rbuf, const int64_t* __restrict__ bf_off,
                                                        int* __restrict__ status) {
  __shared__ double s_row[2][BF_NB], s_col[2][BF_NB];
  const int m = m_first + blockIdx.x;
  const int n = L - m;
  const int nb = min(BF_NB, n - j0);
  const double* A = ainv + __ldg(ainv_off + m);
  const int tid = threadIdx.x;
  // R = A[J, :] for columns of this chunk, layout [col][NB]
  {
    double* R = rbuf + __ldg(bf_off + m);
    const int c0 = blockIdx.y * BF_RCHUNK, c1 = min(n, c0 + BF_RCHUNK);
    const int tot = (c1 - c0) * BF_NB;
    // 8 independent loads in flight per thread before the stores
    for (int base = 0; base < tot; base += 8 * BF_THREADS) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = base + u * BF_THREADS + tid;
        const int r = idx & (BF_NB - 1), c = c0 + (idx >> 6);
        v[u] = (idx < tot && r < nb) ? __ldcg(A + (int64_t)c * n + j0 + r) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = base + u * BF_THREADS + tid;
        if (idx < tot) R[(int64_t)(c0 + (idx >> 6)) * BF_NB + (idx & (BF_NB - 1))] = v[u];
      }
    }
  }
  if (blockIdx.y != 0) return;
  const int tr = tid >> 4, tc = tid & 15;  // patch rows 4tr.., columns 4tc..
  double d[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = 4 * tr + i, c = 4 * tc + j;
      d[i][j] = (r < nb && c < nb) ? __ldcg(A + (int64_t)(j0 + c) * n + j0 + r) : (r == c ? 1.0 : 0.0);
    }
  bool bad = false;
  for (int p = 0; p < nb; ++p) {
    const int buf = p & 1;
    // static register indices only (a runtime index would spill d to local memory)
    const int q = p & 3;
    if ((p >> 2) == tr) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        s_row[buf][4 * tc + j] = q == 0 ? d[0][j] : q == 1 ? d[1][j] : q == 2 ? d[2][j] : d[3][j];
    }
    if ((p >> 2) == tc) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        s_col[buf][4 * tr + i] = q == 0 ? d[i][0] : q == 1 ? d[i][1] : q == 2 ? d[i][2] : d[i][3];
    }
    __syncthreads();
    const double piv = s_row[buf][p];
    const double inv = 1.0 / piv;
    if (tid == 0 && (piv == 0.0 || !isfinite(piv))) bad = true;
    double pc[4], pr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) pc[i] = s_col[buf][4 * tr + i] * inv;
#pragma unroll
    for (int j = 0; j < 4; ++j) pr[j] = s_row[buf][4 * tc + j];
    // branch-free: rows r != p subtract pc * prow, row p scales by 1/piv,
    // column p becomes -pc (its pivot entry 1/piv)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool rp = 4 * tr + i == p;
      const double gi = rp ? 0.0 : pc[i];
      const double si = rp ? inv : 1.0;
      const double colv = rp ? inv : -pc[i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double v = fma(-gi, pr[j], si * d[i][j]);
        d[i][j] = (4 * tc + j == p) ? colv : v;
      }
    }
  }
  if (bad) atomicOr(status + m, 1);
  double* Dg = dbuf + (size_t)blockIdx.x * BF_NB * BF_NB;  // D[r][c] at c * NB + r
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) Dg[(4 * tc + j) * BF_NB + 4 * tr + i] = d[i][j];
}

// ---- 2a'. The same D with a short dependency chain: 64 threads, one row of
// the identity-padded 64 x 64 block per thread in registers, kept ROTATED so
// the current pivot column is always register 0 (static register indices in a
// rolled loop, as factor_np.cu's panel step).  Per pivot the pivot row is
// published with its reciprocal through a double-buffered shared record (one
// 64-thread barrier); every other row subtracts g = d[0] / piv times it; the
// pivot row's own scale is applied at the end.  After 64 steps the rotation is
// back to natural order and the rows are those of D (identity past nb).
__global__ void __launch_bounds__(64) k_bf_diag_rows(int L, int m_first, int j0,
                                                     const int64_t* __restrict__ ainv_off,
                                                     const double* __restrict__ ainv, double* __restrict__ dbuf,
                                                     int* __restrict__ status) {
  __shared__ __align__(16) double rec[2][BF_NB + 2];  // pivot row columns p+1 .. p+63 (rotated), 1 / pivot
  const int m = m_first + blockIdx.x;
  const int n = L - m;
  const int nb = min(BF_NB, n - j0);
  const double* A = ainv + __ldg(ainv_off + m);
  const int r = threadIdx.x;
  double d[BF_NB];
#pragma unroll
  for (int c = 0; c < BF_NB; ++c)
    d[c] = (r < nb && c < nb) ? __ldcg(A + (int64_t)(j0 + c) * n + j0 + r) : (r == c ? 1.0 : 0.0);
  bool bad = false;
  // rinv = 1 / d[0], computed by every row as soon as its new d[0] exists so
  // the division's latency hides under the row update (only row p + 1 uses it)
  auto publish = [&](double* pn, double rinv) {
#pragma unroll
    for (int c = 0; c < BF_NB - 2; c += 2) *reinterpret_cast<double2*>(pn + c) = make_double2(d[c + 1], d[c + 2]);
    if (d[0] == 0.0 || !isfinite(d[0])) bad = true;
    *reinterpret_cast<double2*>(pn + BF_NB - 2) = make_double2(d[BF_NB - 1], rinv);
  };
  double rsc = 1.0;
  if (r == 0) publish(rec[0], 1.0 / d[0]);
#pragma unroll 1
  for (int p = 0; p < BF_NB; ++p) {
    __syncthreads();
    const double* pr = rec[p & 1];
    const double inv = pr[BF_NB - 1];
    const bool ispiv = r == p;
    const double gg = ispiv ? 0.0 : d[0] * inv;
    rsc = ispiv ? inv : rsc;
    const double2 v0 = *reinterpret_cast<const double2*>(pr);
    d[0] = fma(-gg, v0.x, d[1]);
    const double rinv = 1.0 / d[0];
    d[1] = fma(-gg, v0.y, d[2]);
#pragma unroll
    for (int c = 2; c < BF_NB - 1; c += 2) {
      const double2 v = *reinterpret_cast<const double2*>(pr + c);
      d[c] = fma(-gg, v.x, d[c + 1]);
      if (c + 1 < BF_NB - 1) d[c + 1] = fma(-gg, v.y, d[c + 2]);
    }
    d[BF_NB - 1] = ispiv ? 1.0 : -gg;
    if (r == p + 1) publish(rec[(p + 1) & 1], rinv);
  }
  if (bad) atomicOr(status + m, 1);
  double* Dg = dbuf + (size_t)blockIdx.x * BF_NB * BF_NB;  // D[r][c] at c * NB + r
#pragma unroll
  for (int c = 0; c < BF_NB; ++c) Dg[c * BF_NB + r] = d[c] * rsc;
}

// R = A[J, :] (the update's B operand), layout [col][NB]; grid (orders, column chunks).
__global__ void __launch_bounds__(BF_THREADS) k_bf_rcopy(int L, int m_first, int j0,
                                                         const int64_t* __restrict__ ainv_off,
                                                         const double* __restrict__ ainv, double* __restrict__ rbuf,
                                                         const int64_t* __restrict__ bf_off) {
  const int m = m_first + blockIdx.x;
  const int n = L - m;
  const int nb = min(BF_NB, n - j0);
  const double* A = ainv + __ldg(ainv_off + m);
  double* R = rbuf + __ldg(bf_off + m);
  const int c0 = blockIdx.y * BF_RCHUNK, c1 = min(n, c0 + BF_RCHUNK);
  const int tot = (c1 - c0) * BF_NB;
  for (int base = 0; base < tot; base += 8 * BF_THREADS) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * BF_THREADS + threadIdx.x;
      const int rr = idx & (BF_NB - 1), c = c0 + (idx >> 6);
      v[u] = (idx < tot && rr < nb) ? __ldcg(A + (int64_t)c * n + j0 + rr) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * BF_THREADS + threadIdx.x;
      if (idx < tot) R[(int64_t)(c0 + (idx >> 6)) * BF_NB + (idx & (BF_NB - 1))] = v[u];
    }
  }
}

// ---- 2b. E = -A[I, J] D (E[J] = D - I) per 64-row tile; A[I, J] = E + I_J.
__global__ void __launch_bounds__(BF_THREADS) k_bf_panel(int L, int m_first, int j0, const int* __restrict__ pre,
                                                         int cnt, const int64_t* __restrict__ ainv_off,
                                                         double* __restrict__ ainv, const double* __restrict__ dbuf,
                                                         double* __restrict__ ebuf, const int64_t* __restrict__ bf_off) {
  extern __shared__ double bf_sm[];
  double(*At)[BF_LDS] = reinterpret_cast<double(*)[BF_LDS]>(bf_sm);                 // [k][row]
  double(*Ds)[BF_LDS] = reinterpret_cast<double(*)[BF_LDS]>(bf_sm + BF_NB * BF_LDS);  // [k][c]
  __shared__ int s_oi;
  if (threadIdx.x < 32) {
    const int oi_w = bf_find_warp(pre, cnt, blockIdx.x);
    if (threadIdx.x == 0) s_oi = oi_w;
  }
  __syncthreads();
  const int oi = s_oi;
  const int m = m_first + oi;
  const int n = L - m, lde = bf_lde(n);
  const int nb = min(BF_NB, n - j0);
  const int i0 = (blockIdx.x - __ldg(pre + oi)) * BF_T;
  double* A = ainv + __ldg(ainv_off + m);
  const double* Dg = dbuf + (size_t)oi * BF_NB * BF_NB;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < BF_T * BF_NB; idx += BF_THREADS) {
    const int r = idx & (BF_T - 1), c = idx >> 6;
    At[c][r] = (i0 + r < n && c < nb) ? __ldcg(A + (int64_t)(j0 + c) * n + i0 + r) : 0.0;
    Ds[c][r] = __ldcg(Dg + idx);  // D[r][c] is stored at c * NB + r
  }
  __syncthreads();
  double* E = ebuf + __ldg(bf_off + m);  // [col][lde]
  const int r = tid & (BF_T - 1), cg4 = tid >> 6;  // row r, columns cg4*16 .. +16
  const int gi = i0 + r;
  const bool inJ = gi >= j0 && gi < j0 + nb;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  if (!inJ) {
#pragma unroll 4
    for (int k = 0; k < BF_NB; ++k) {
      const double a = At[k][r];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = fma(a, Ds[cg4 * 16 + q][k], acc[q]);
    }
  }
  if (gi < n) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int c = cg4 * 16 + q;
      if (c >= nb) continue;
      const double v = inJ ? Ds[c][gi - j0] - ((gi - j0 == c) ? 1.0 : 0.0) : -acc[q];
      E[(int64_t)c * lde + gi] = v;
      A[(int64_t)(j0 + c) * n + gi] = v + ((inJ && gi - j0 == c) ? 1.0 : 0.0);
    }
  }
}

// ---- 2b'. The panel on the tensor cores: one 64-row tile per CTA computes
// A[I, J] D (64 x 64 x 64, DMMA, operands in shared memory: A[I, J] k-major,
// D column-major as stored), then E = -A[I, J] D (E[J] = D - I) and
// A[I, J] = E + I_J as k_bf_panel does.
__global__ void __launch_bounds__(BF_THREADS, 3) k_bf_panel_mma(int L, int m_first, int j0, const int* __restrict__ pre,
                                                                int cnt, const int64_t* __restrict__ ainv_off,
                                                                double* __restrict__ ainv,
                                                                const double* __restrict__ dbuf,
                                                                double* __restrict__ ebuf,
                                                                const int64_t* __restrict__ bf_off,
                                                                double* __restrict__ rnext) {
  extern __shared__ __align__(16) double bf_sm[];
  double(*At)[BF_LDS] = reinterpret_cast<double(*)[BF_LDS]>(bf_sm);                 // [k][row]
  double(*Dt)[BF_LDS] = reinterpret_cast<double(*)[BF_LDS]>(bf_sm + BF_NB * BF_LDS);  // [c][k] = D[k][c]
  __shared__ int s_oi;
  if (threadIdx.x < 32) {
    const int oi_w = bf_find_warp(pre, cnt, blockIdx.x);
    if (threadIdx.x == 0) s_oi = oi_w;
  }
  __syncthreads();
  const int oi = s_oi;
  const int m = m_first + oi;
  const int n = L - m, lde = bf_lde(n);
  const int nb = min(BF_NB, n - j0);
  const int i0 = (blockIdx.x - __ldg(pre + oi)) * BF_T;
  double* A = ainv + __ldg(ainv_off + m);
  const double* Dg = dbuf + (size_t)oi * BF_NB * BF_NB;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < BF_NB * BF_NB / 2; idx += BF_THREADS) {  // D: column c, k2, k2 + 1
    const int c = idx >> 5, k2 = (idx & 31) * 2;
    bf_cp16(&Dt[c][k2], Dg + c * BF_NB + k2);
  }
  for (int idx = tid; idx < BF_T * BF_NB; idx += BF_THREADS) {  // A[I, J]: column k, row r
    const int r = idx & (BF_T - 1), k = idx >> 6;
    At[k][r] = (i0 + r < n && k < nb) ? __ldcg(A + (int64_t)(j0 + k) * n + i0 + r) : 0.0;
  }
  bf_cp_wait_all();
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = (warp & 1) * 32, wc = (warp >> 1) * 16;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < BF_NB; k0 += 4) {
    double a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = At[k0 + t][wr + 8 * i + g];
#pragma unroll
    for (int j = 0; j < 2; ++j) b[j] = Dt[wc + 8 * j + g][k0 + t];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
  double* E = ebuf + __ldg(bf_off + m);  // [col][lde]
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = i0 + wr + 8 * i + g;
    if (row >= n) continue;
    const bool inJ = row >= j0 && row < j0 + nb;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = wc + 8 * j + 2 * t + h;
        if (c >= nb) continue;
        const bool diag = inJ && row - j0 == c;
        const double v = inJ ? Dt[c][row - j0] - (diag ? 1.0 : 0.0) : -acc[i][j][h];
        E[(int64_t)c * lde + row] = v;
        A[(int64_t)(j0 + c) * n + row] = v + (diag ? 1.0 : 0.0);
        // next step's R = A[J', :] (J' = the next 64 rows): its J columns are final here
        if (rnext && row >= j0 + BF_NB && row < j0 + 2 * BF_NB)
          rnext[__ldg(bf_off + m) + (int64_t)(j0 + c) * BF_NB + (row - j0 - BF_NB)] = v;
      }
  }
}

// ---- 2c. A[I, K] += E[I, :] R[:, K] for every 64 x 64 tile outside column block J.
// E and R are staged by 16-byte async copies (k-major / column-major in smem,
// matching their global layouts) while the C fragments load from global.
__global__ void __launch_bounds__(BF_THREADS, 3) k_bf_update(int L, int m_first, int j0, const int* __restrict__ pre,
                                                             int cnt, const int64_t* __restrict__ ainv_off,
                                                             double* __restrict__ ainv, const double* __restrict__ ebuf,
                                                             const double* __restrict__ rbuf,
                                                             const int64_t* __restrict__ bf_off,
                                                             double* __restrict__ rnext) {
  extern __shared__ __align__(16) double bf_sm[];
  double(*Et)[BF_LDS] = reinterpret_cast<double(*)[BF_LDS]>(bf_sm);                 // [k][row]
  double(*Rt)[BF_LDS] = reinterpret_cast<double(*)[BF_LDS]>(bf_sm + BF_NB * BF_LDS);  // [col][k]
  __shared__ int s_oi;
  if (threadIdx.x < 32) {
    const int oi_w = bf_find_warp(pre, cnt, blockIdx.x);
    if (threadIdx.x == 0) s_oi = oi_w;
  }
  __syncthreads();
  const int oi = s_oi;
  const int m = m_first + oi;
  const int n = L - m, lde = bf_lde(n);
  const int nb = min(BF_NB, n - j0);
  const int nt = (n + BF_T - 1) / BF_T;
  const int local = blockIdx.x - __ldg(pre + oi);
  const int rt = local % nt;
  int ct = local / nt;
  if (ct >= j0 / BF_T) ++ct;  // skip the panel's column tile
  const int i0 = rt * BF_T, c0 = ct * BF_T;
  double* A = ainv + __ldg(ainv_off + m);
  const double* E = ebuf + __ldg(bf_off + m);
  const double* R = rbuf + __ldg(bf_off + m);
  const int tid = threadIdx.x;
  // async staging: 64 x 64 doubles each = 2048 16-byte chunks, 8 per thread per operand
  for (int idx = tid; idx < BF_T * BF_NB / 2; idx += BF_THREADS) {
    const int k = idx >> 5, r2 = (idx & 31) * 2;  // E: column k, rows r2, r2+1
    if (k < nb && i0 + r2 + 1 < lde) bf_cp16(&Et[k][r2], E + (int64_t)k * lde + i0 + r2);
    else {
      Et[k][r2] = 0.0;
      Et[k][r2 + 1] = 0.0;
    }
    const int c = idx >> 5, k2 = (idx & 31) * 2;  // R: column c0 + c, k2, k2+1
    if (c0 + c < n) bf_cp16(&Rt[c][k2], R + (int64_t)(c0 + c) * BF_NB + k2);
    else {
      Rt[c][k2] = 0.0;
      Rt[c][k2 + 1] = 0.0;
    }
  }
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = (warp & 1) * 32, wc = (warp >> 1) * 16;  // warp tile 32 rows x 16 cols
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int row = i0 + wr + 8 * i + g, col = c0 + wc + 8 * j + 2 * t;
      acc[i][j][0] = (row < n && col < n) ? __ldcg(A + (int64_t)col * n + row) : 0.0;
      acc[i][j][1] = (row < n && col + 1 < n) ? __ldcg(A + (int64_t)(col + 1) * n + row) : 0.0;
    }
  bf_cp_wait_all();
  __syncthreads();
  // rows of E beyond n (padding) are zero in E only if i0 + r < n: mask them here
#pragma unroll 4
  for (int k0 = 0; k0 < BF_NB; k0 += 4) {
    double a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = Et[k0 + t][wr + 8 * i + g];
#pragma unroll
    for (int j = 0; j < 2; ++j) b[j] = Rt[wc + 8 * j + g][k0 + t];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int row = i0 + wr + 8 * i + g, col = c0 + wc + 8 * j + 2 * t;
      if (row < n && col < n) A[(int64_t)col * n + row] = acc[i][j][0];
      if (row < n && col + 1 < n) A[(int64_t)(col + 1) * n + row] = acc[i][j][1];
      if (rnext && i0 == j0 + BF_T && row < n) {  // the next step's R = A[J', :] from the J' row tile
        double* Rn = rnext + __ldg(bf_off + m);
        if (col < n) Rn[(int64_t)col * BF_NB + (row - i0)] = acc[i][j][0];
        if (col + 1 < n) Rn[(int64_t)(col + 1) * BF_NB + (row - i0)] = acc[i][j][1];
      }
    }
}

// ---- 2c (wide). The same update on 128 x 64 tiles: eight warps of 32 x 32,
// so each k-step loads 8 fragments for 16 DMMAs (the 64 x 64 tile: 6 for 8)
// and every E / R element staged in shared memory feeds twice the math.
// 101 KB of shared memory, two CTAs per SM.  Default for L >= 1024
// (OSPH_BF_UPD_ROWS=64|128 forces either kernel).
#define BF_TW 128
#define BF_LDW (BF_TW + 4)
__global__ void __launch_bounds__(BF_THREADS, 2) k_bf_update_w(int L, int m_first, int j0, const int* __restrict__ pre,
                                                               int cnt, const int64_t* __restrict__ ainv_off,
                                                               double* __restrict__ ainv, const double* __restrict__ ebuf,
                                                               const double* __restrict__ rbuf,
                                                               const int64_t* __restrict__ bf_off,
                                                               double* __restrict__ rnext) {
  extern __shared__ __align__(16) double bf_sm[];
  double(*Et)[BF_LDW] = reinterpret_cast<double(*)[BF_LDW]>(bf_sm);                  // [k][row]
  double(*Rt)[BF_LDS] = reinterpret_cast<double(*)[BF_LDS]>(bf_sm + BF_NB * BF_LDW);  // [col][k]
  __shared__ int s_oi;
  if (threadIdx.x < 32) {
    const int oi_w = bf_find_warp(pre, cnt, blockIdx.x);
    if (threadIdx.x == 0) s_oi = oi_w;
  }
  __syncthreads();
  const int oi = s_oi;
  const int m = m_first + oi;
  const int n = L - m, lde = bf_lde(n);
  const int nb = min(BF_NB, n - j0);
  const int nt = (n + BF_TW - 1) / BF_TW;
  const int local = blockIdx.x - __ldg(pre + oi);
  const int rt = local % nt;
  int ct = local / nt;
  if (ct >= j0 / BF_T) ++ct;  // skip the panel's column tile
  const int i0 = rt * BF_TW, c0 = ct * BF_T;
  double* A = ainv + __ldg(ainv_off + m);
  const double* E = ebuf + __ldg(bf_off + m);
  const double* R = rbuf + __ldg(bf_off + m);
  const int tid = threadIdx.x;
  for (int idx = tid; idx < BF_TW * BF_NB / 2; idx += BF_THREADS) {
    const int k = idx >> 6, r2 = (idx & 63) * 2;  // E: column k, rows r2, r2+1
    if (k < nb && i0 + r2 + 1 < lde) bf_cp16(&Et[k][r2], E + (int64_t)k * lde + i0 + r2);
    else {
      Et[k][r2] = 0.0;
      Et[k][r2 + 1] = 0.0;
    }
  }
  for (int idx = tid; idx < BF_T * BF_NB / 2; idx += BF_THREADS) {
    const int c = idx >> 5, k2 = (idx & 31) * 2;  // R: column c0 + c, k2, k2+1
    if (c0 + c < n) bf_cp16(&Rt[c][k2], R + (int64_t)(c0 + c) * BF_NB + k2);
    else {
      Rt[c][k2] = 0.0;
      Rt[c][k2 + 1] = 0.0;
    }
  }
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = (warp & 3) * 32, wc = (warp >> 2) * 32;  // warp tile 32 rows x 32 cols
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = i0 + wr + 8 * i + g, col = c0 + wc + 8 * j + 2 * t;
      acc[i][j][0] = (row < n && col < n) ? __ldcg(A + (int64_t)col * n + row) : 0.0;
      acc[i][j][1] = (row < n && col + 1 < n) ? __ldcg(A + (int64_t)(col + 1) * n + row) : 0.0;
    }
  bf_cp_wait_all();
  __syncthreads();
#pragma unroll 2
  for (int k0 = 0; k0 < BF_NB; k0 += 4) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = Et[k0 + t][wr + 8 * i + g];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = Rt[wc + 8 * j + g][k0 + t];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
  double* Rn = rnext ? rnext + __ldg(bf_off + m) : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = i0 + wr + 8 * i + g, col = c0 + wc + 8 * j + 2 * t;
      if (row < n && col < n) A[(int64_t)col * n + row] = acc[i][j][0];
      if (row < n && col + 1 < n) A[(int64_t)(col + 1) * n + row] = acc[i][j][1];
      // the next step's R = A[J', :] (rows j0 + 64 .. j0 + 127; never split across 128-row tiles)
      if (Rn && row >= j0 + BF_NB && row < j0 + 2 * BF_NB && row < n) {
        if (col < n) Rn[(int64_t)col * BF_NB + (row - j0 - BF_NB)] = acc[i][j][0];
        if (col + 1 < n) Rn[(int64_t)(col + 1) * BF_NB + (row - j0 - BF_NB)] = acc[i][j][1];
      }
    }
}

// ---- 2c'. Persistent, software-pipelined variant of the update: one CTA per
// SM walks a contiguous range of work items (consecutive items share the
// order, so the item -> order mapping advances incrementally instead of being
// searched), and while it multiplies item i out of shared memory the
// 16-/8-byte async copies of item i+1's E, R and C tiles are in flight.  Two
// stages of (E, R, C) = 207 KB of shared memory.  Opt-in (OSPH_BF_PERSISTENT=1):
// slower than three independent CTAs per SM at L = 2048 (691 vs 549 ms).
#define BF_LDC (BF_T + 2)
struct BfStageP {
  double e[BF_NB][BF_LDS];  // [k][row]
  double r[BF_T][BF_LDS];   // [col][k]
  double c[BF_T][BF_LDC];   // [col][row]
};
__device__ __forceinline__ void bf_cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(bf_smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void bf_cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void bf_cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

__global__ void __launch_bounds__(BF_THREADS, 1) k_bf_update_p(int L, int m_first, int j0, const int* __restrict__ pre,
                                                               int cnt, int total, const int64_t* __restrict__ ainv_off,
                                                               double* __restrict__ ainv,
                                                               const double* __restrict__ ebuf,
                                                               const double* __restrict__ rbuf,
                                                               const int64_t* __restrict__ bf_off) {
  extern __shared__ __align__(16) unsigned char bfp_raw[];
  BfStageP* stg = reinterpret_cast<BfStageP*>(bfp_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int it0 = blockIdx.x * per, it1 = min(total, it0 + per);
  if (it0 >= it1) return;
  __shared__ int s_oi0;
  if (warp == 0) {
    const int o = bf_find_warp(pre, cnt, it0);
    if (lane == 0) s_oi0 = o;
  }
  __syncthreads();
  // item cursor (identical in every thread)
  int oi = s_oi0, base = __ldg(pre + oi), next = __ldg(pre + oi + 1);
  auto item = [&](int it, int& m, int& n, int& i0, int& c0) {
    while (it >= next) {
      ++oi;
      base = next;
      next = __ldg(pre + oi + 1);
    }
    m = m_first + oi;
    n = L - m;
    const int nt = (n + BF_T - 1) / BF_T;
    const int local = it - base;
    int ct = local / nt;
    if (ct >= j0 / BF_T) ++ct;
    i0 = (local % nt) * BF_T;
    c0 = ct * BF_T;
  };
  auto issue = [&](BfStageP& S, int m, int n, int i0, int c0) {
    const int lde = bf_lde(n), nb = min(BF_NB, n - j0);
    const double* A = ainv + __ldg(ainv_off + m);
    const double* E = ebuf + __ldg(bf_off + m);
    const double* R = rbuf + __ldg(bf_off + m);
    for (int idx = tid; idx < BF_T * BF_NB / 2; idx += BF_THREADS) {
      const int k = idx >> 5, r2 = (idx & 31) * 2;  // E: column k, rows r2, r2 + 1
      if (k < nb && i0 + r2 + 1 < lde) bf_cp16(&S.e[k][r2], E + (int64_t)k * lde + i0 + r2);
      else {
        S.e[k][r2] = 0.0;
        S.e[k][r2 + 1] = 0.0;
      }
      const int c = idx >> 5, k2 = (idx & 31) * 2;  // R: column c0 + c, k2, k2 + 1
      if (c0 + c < n) bf_cp16(&S.r[c][k2], R + (int64_t)(c0 + c) * BF_NB + k2);
      else {
        S.r[c][k2] = 0.0;
        S.r[c][k2 + 1] = 0.0;
      }
    }
    for (int idx = tid; idx < BF_T * BF_T; idx += BF_THREADS) {  // C: column c0 + c, row i0 + r (8-byte pieces)
      const int c = idx >> 6, r = idx & 63;
      if (i0 + r < n && c0 + c < n) bf_cp8(&S.c[c][r], A + (int64_t)(c0 + c) * n + i0 + r);
      else S.c[c][r] = 0.0;
    }
    bf_cp_commit();
  };
  const int wr = (warp & 1) * 32, wc = (warp >> 1) * 16;
  int m, n, i0, c0;
  item(it0, m, n, i0, c0);
  issue(stg[0], m, n, i0, c0);
  for (int it = it0; it < it1; ++it) {
    const int cm = m, cn = n, ci0 = i0, cc0 = c0;
    if (it + 1 < it1) {
      item(it + 1, m, n, i0, c0);
      issue(stg[(it + 1 - it0) & 1], m, n, i0, c0);
      bf_cp_wait1();
    } else {
      bf_cp_wait_all();
    }
    __syncthreads();
    const BfStageP& S = stg[(it - it0) & 1];
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = wr + 8 * i + g, c = wc + 8 * j + 2 * t;
        acc[i][j][0] = S.c[c][r];
        acc[i][j][1] = S.c[c + 1][r];
      }
#pragma unroll 4
    for (int k0 = 0; k0 < BF_NB; k0 += 4) {
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = S.e[k0 + t][wr + 8 * i + g];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = S.r[wc + 8 * j + g][k0 + t];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    double* A = ainv + __ldg(ainv_off + cm);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int row = ci0 + wr + 8 * i + g, col = cc0 + wc + 8 * j + 2 * t;
        if (row < cn && col < cn) A[(int64_t)col * cn + row] = acc[i][j][0];
        if (row < cn && col + 1 < cn) A[(int64_t)(col + 1) * cn + row] = acc[i][j][1];
      }
    __syncthreads();  // stage (it - it0) & 1 is refilled by the next iteration's issue
  }
}

// ---- 3. sweep operands from X (column c = pivot position, ring perm[c]):
// chunk-major tiles with natural-order columns (the late ring's column zero),
// u_m[perm[c]] = Pb_m[m-1, :] X[:, c], and for c = j* (perm = 0): w_m, beta_m, j*.
__global__ void __launch_bounds__(BF_THREADS) k_bf_epilogue(int L, int m_first, const int64_t* __restrict__ ainv_off,
                                                            const double* __restrict__ ainv,
                                                            const int* __restrict__ perm_all,
                                                            const int64_t* __restrict__ xt_off,
                                                            double* __restrict__ xt_all,
                                                            const int64_t* __restrict__ pb_off,
                                                            const double* __restrict__ pbelow, double* __restrict__ u_out,
                                                            double* __restrict__ w_out, double* __restrict__ beta_out,
                                                            int* __restrict__ jstar_out) {
  const int m = m_first + blockIdx.y;
  const int n = L - m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* A = ainv + __ldg(ainv_off + m);
  const int* perm = perm_all + packed_pos(L, m, 0);
  double* Xt = xt_all + __ldg(xt_off + m);
  const double* Pb = pbelow + __ldg(pb_off + m);
  const int nrt = (n + 7) >> 3, nrtpb = (m + 7) >> 3;
  for (int c = blockIdx.x * (BF_THREADS / 32) + warp; c < n; c += gridDim.x * (BF_THREADS / 32)) {
    const int cn = __ldg(perm + c);
    const double* col = A + (int64_t)c * n;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) {
      const double v = __ldcg(col + i);
      Xt[tile_index(i, cn, nrt)] = cn != 0 ? v : 0.0;
      if (m >= 1) s = fma(__ldcg(Pb + tile_index(m - 1, i, nrtpb)), v, s);
      if (cn == 0) w_out[(size_t)m * uw_ld(L) + i] = v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      u_out[(size_t)m * uw_ld(L) + cn] = cn != 0 ? s : 0.0;
      if (cn == 0) {
        beta_out[m] = s;
        jstar_out[m] = c;
      }
    }
  }
}

// ---- host side ------------------------------------------------------------

// E / R panel storage of one order (doubles), for offset tables built by the plan.
int64_t bf_panel_doubles(int n) { return (int64_t)BF_NB * bf_lde(n); }
int64_t bf_diag_doubles(int orders) { return (int64_t)BF_NB * BF_NB * orders; }

// Step tables of work items for orders m_first..m_last (built once per range).
cudaError_t bf_prepare(osph_plan* p, int m_first, int m_last, BfRange* r) {
  const int L = p->L;
  const int nmax = L - m_first;
  const int nsteps = (nmax + BF_NB - 1) / BF_NB;
  std::vector<int> tab;
  r->m_first = m_first;
  r->m_last = m_last;
  r->steps.assign(nsteps, {});
  for (int sidx = 0; sidx < nsteps; ++sidx) {
    const int j0 = sidx * BF_NB;
    int cnt = 0;
    for (int m = m_first; m <= m_last; ++m)
      if (L - m > j0) cnt = m - m_first + 1;
    auto& d = r->steps[sidx];
    d.cnt = cnt;
    d.pre_panel = (int)tab.size();
    int acc = 0;
    for (int o = 0; o <= cnt; ++o) {
      tab.push_back(acc);
      if (o < cnt) acc += (L - (m_first + o) + BF_T - 1) / BF_T;
    }
    d.n_panel = acc;
    d.pre_upd = (int)tab.size();
    acc = 0;
    for (int o = 0; o <= cnt; ++o) {
      tab.push_back(acc);
      if (o < cnt) {
        const int nt = (L - (m_first + o) + BF_T - 1) / BF_T;
        acc += nt * (nt - 1);
      }
    }
    d.n_upd = acc;
    d.pre_updw = (int)tab.size();
    acc = 0;
    for (int o = 0; o <= cnt; ++o) {
      tab.push_back(acc);
      if (o < cnt) {
        const int n = L - (m_first + o);
        acc += ((n + BF_TW - 1) / BF_TW) * ((n + BF_T - 1) / BF_T - 1);
      }
    }
    d.n_updw = acc;
  }
  cudaError_t e;
  cudaFree(r->d_tab);
  r->d_tab = nullptr;
  if ((e = cudaMalloc(&r->d_tab, sizeof(int) * tab.size())) != cudaSuccess) return e;
  return cudaMemcpy(r->d_tab, tab.data(), sizeof(int) * tab.size(), cudaMemcpyHostToDevice);
}

// Factor orders r.m_first..r.m_last with the recorded pivot order, writing A/X,
// Pb, the tiled X and the sweep constants at the given offset tables.
cudaError_t bf_run(osph_plan* p, const BfRange& r, cudaStream_t st, const BfOffsets& o) {
  const int L = p->L;
  const int m_first = r.m_first;
  const int cnt_all = r.m_last - r.m_first + 1;
  cudaError_t e;
  const size_t sm2 = sizeof(double) * 2 * BF_T * BF_LDS + 16;
  if ((e = cudaFuncSetAttribute(k_bf_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_bf_panel_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2)) !=
      cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_bf_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2)) != cudaSuccess)
    return e;
  const size_t smw = sizeof(double) * (BF_NB * BF_LDW + BF_T * BF_LDS) + 16;
  if ((e = cudaFuncSetAttribute(k_bf_update_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw)) !=
      cudaSuccess)
    return e;
  // 128-row tiles win at large L (config 4: 1.574 vs 1.564 transforms/s), 64-row ones at L = 256
  // (config 2: 32.5k vs 32.3k); OSPH_BF_UPD_ROWS=64|128 forces one
  static const int upd_rows_env = getenv("OSPH_BF_UPD_ROWS") ? atoi(getenv("OSPH_BF_UPD_ROWS")) : 0;
  const bool upd_wide = upd_rows_env ? upd_rows_env == 128 : L >= 1024;
  if ((e = cudaFuncSetAttribute(k_bf_update_p, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(BfStageP) * 2))) != cudaSuccess)
    return e;
  if (p->num_sms == 0) {
    cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device);
    // measured at L = 2048: 691 ms persistent vs 549 ms one CTA per tile (3 CTAs/SM hide latency better)
    p->bf_persistent = getenv("OSPH_BF_PERSISTENT") ? atoi(getenv("OSPH_BF_PERSISTENT")) != 0 : false;
  }
  k_bf_generate<<<dim3((L + BF_THREADS - 1) / BF_THREADS, cnt_all), BF_THREADS, 0, st>>>(
      L, m_first, p->d_cos, p->d_rec, p->d_ls, p->d_pstart, p->d_piv, o.ainv, o.pb, p->d_ainv, p->d_pbelow);
  if (p->d_at) {  // the blocks themselves for the sweep's refinement step, natural ring order
    k_bf_generate_at<<<dim3((L + BF_THREADS - 1) / BF_THREADS, cnt_all), BF_THREADS, 0, st>>>(
        L, m_first, p->d_cos, p->d_rec, p->d_ls, p->d_pstart, o.xt, p->d_at);
    p->launches++;
  }
  p->launches++;
  if (p->need_norms) {  // ||A||_1 and ||X||_1 feed only the check=True condition estimate
    k_bf_colnorm<<<dim3(8, cnt_all), BF_THREADS, 0, st>>>(L, m_first, o.ainv, p->d_ainv, p->d_norms, 0);
    p->launches++;
  }
  for (size_t sidx = 0; sidx < r.steps.size(); ++sidx) {
    const auto& d = r.steps[sidx];
    const int j0 = (int)sidx * BF_NB;
    const dim3 dgrid(d.cnt, (L - m_first + BF_RCHUNK - 1) / BF_RCHUNK);
    // R = A[J, :] of this step: copied at step 0; afterwards written by the
    // previous step's panel (J columns) and update (J-row tiles) into the
    // other of two buffers (the variants below copy it every step instead)
    static const bool rfuse_env = !(getenv("OSPH_BF_RFUSE") && atoi(getenv("OSPH_BF_RFUSE")) == 0);
    const bool fused_r = rfuse_env && !getenv("OSPH_BF_DIAG_PATCH") && !getenv("OSPH_BF_PANEL_FMA") && !p->bf_persistent;
    double* rcur = p->d_bf_r + (fused_r ? (int64_t)(sidx & 1) * p->bf_r_half : 0);
    double* rnext = fused_r ? p->d_bf_r + (int64_t)((sidx + 1) & 1) * p->bf_r_half : nullptr;
    if (!getenv("OSPH_BF_DIAG_PATCH")) {  // register-row diagonal inverse (+ R copy when needed)
      if (sidx == 0 || !fused_r) {
        k_bf_rcopy<<<dgrid, BF_THREADS, 0, st>>>(L, m_first, j0, o.ainv, p->d_ainv, rcur, o.bf);
        p->launches++;
      }
      k_bf_diag_rows<<<d.cnt, 64, 0, st>>>(L, m_first, j0, o.ainv, p->d_ainv, p->d_bf_d, p->d_status);
      p->launches++;
    } else {  // 4 x 4 register patch per thread, R copied by the same kernel
      k_bf_diag<<<dgrid, BF_THREADS, 0, st>>>(L, m_first, j0, o.ainv, p->d_ainv, p->d_bf_d, rcur, o.bf,
                                              p->d_status);
      p->launches++;
    }
    if (!getenv("OSPH_BF_PANEL_FMA"))
      k_bf_panel_mma<<<d.n_panel, BF_THREADS, sm2, st>>>(L, m_first, j0, r.d_tab + d.pre_panel, d.cnt, o.ainv,
                                                       p->d_ainv, p->d_bf_d, p->d_bf_e, o.bf, rnext);
    else
      k_bf_panel<<<d.n_panel, BF_THREADS, sm2, st>>>(L, m_first, j0, r.d_tab + d.pre_panel, d.cnt, o.ainv,
                                                   p->d_ainv, p->d_bf_d, p->d_bf_e, o.bf);
    p->launches++;
    if (d.n_upd > 0 && p->bf_persistent) {
      const int ctas = std::min(d.n_upd, p->num_sms);
      k_bf_update_p<<<ctas, BF_THREADS, sizeof(BfStageP) * 2, st>>>(L, m_first, j0, r.d_tab + d.pre_upd, d.cnt,
                                                                   d.n_upd, o.ainv, p->d_ainv, p->d_bf_e, rcur,
                                                                   o.bf);
    } else if (d.n_upd > 0 && upd_wide)
      k_bf_update_w<<<d.n_updw, BF_THREADS, smw, st>>>(L, m_first, j0, r.d_tab + d.pre_updw, d.cnt, o.ainv,
                                                      p->d_ainv, p->d_bf_e, rcur, o.bf, rnext);
    else if (d.n_upd > 0)
      k_bf_update<<<d.n_upd, BF_THREADS, sm2, st>>>(L, m_first, j0, r.d_tab + d.pre_upd, d.cnt, o.ainv, p->d_ainv,
                                                  p->d_bf_e, rcur, o.bf, rnext);
    if (d.n_upd > 0) p->launches++;
  }
  if (p->need_norms) {
    k_bf_colnorm<<<dim3(8, cnt_all), BF_THREADS, 0, st>>>(L, m_first, o.ainv, p->d_ainv, p->d_norms, 1);
    p->launches++;
  }
  k_bf_epilogue<<<dim3(8, cnt_all), BF_THREADS, 0, st>>>(L, m_first, o.ainv, p->d_ainv, p->d_piv, o.xt, p->d_xt,
                                                         o.pb, p->d_pbelow, p->d_u, p->d_w, p->d_beta, p->d_jstar);
  p->launches++;
  return cudaGetLastError();
}

// The non-windowed plan: every order with n > 256 (m <= L - 257), full offset tables.
cudaError_t launch_factor_bf(osph_plan* p, int m_first, int m_last, cudaStream_t st) {
  cudaError_t e;
  if (p->bf_full.m_first != m_first || p->bf_full.m_last != m_last)
    if ((e = bf_prepare(p, m_first, m_last, &p->bf_full)) != cudaSuccess) return e;
  const BfOffsets o{p->d_ainv_off, p->d_xt_off, p->d_pb_off, p->d_bf_off};
  return bf_run(p, p->bf_full, st, o);
}
