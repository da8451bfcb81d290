// factor_bf.cu -- batched, breadth-first blocked Gauss-Jordan inversion of
// every per-order block with the grid-determined pivot order.
//
// Explicit X = (P A_m)^{-1}, A_m = 2pi Y_lm(theta_k), k >= m, l >= m
// (transform.py:416-429, blocks.py:88-116), organised for throughput instead
// of per-order latency.  With the pivot order known (found once per grid by
// pivots.cu, which runs these same kernels with a partial-pivoting search in
// front of every panel step), row i of the working matrix is ring
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
// epilogue emits the sweep operands (X in
// chunk-major 8-row tiles with natural-order columns, w_m, u_m, j*, beta_m)
// plus ||X||_1 for the condition estimate.
#include <algorithm>
#include <cstdlib>
#include <tuple>
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


#define BF_RCHUNK 256  // columns per R-copy block

// ---- 2a. D = A[J, J]^{-1} (in-place Gauss-Jordan, no interchanges): 64 threads, one row of
// the identity-padded 64 x 64 block per thread in registers, kept ROTATED so
// the current pivot column is always register 0 (static register indices in a
// rolled loop).  Per pivot the pivot row is
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

// ---- 2b. The panel on the tensor cores: one 64-row tile per CTA computes
// A[I, J] D (64 x 64 x 64, DMMA, operands in shared memory: A[I, J] k-major,
// D column-major as stored), then E = -A[I, J] D (E[J] = D - I) and
// A[I, J] = E + I_J.
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

// ---- 2c. The rank-64 (or paired rank-128) trailing update A[I, K] += E R[:, K].
//
// Arguments of the update kernels.  Modes of k_bf_update (64 x 64 tiles):
//   normal      every tile outside the panel's column block(s): rt, ct from the work item;
//   ct_fixed    one column tile, every row tile (the paired step's narrow updates);
//   rt_fixed    one row tile, every column tile outside J1 and J2, the result also
//               copied to rnext (the paired step's R2 = A[J2, :]).
// PAIR: the two panels of a paired step (J1 = [j0, j0 + 64), J2 = [j0 + 64,
// j0 + 128)) in one pass over C: C += E1' R1 + E2 R2, K = 128 in two staged
// halves, with the J2 rows of E1 masked (rows J2 of C already hold A[J2, K] + E1[J2] R1).
struct BfUpdArgs {
  int L, m_first, j0;
  const int* pre;
  int cnt;
  const int64_t* ainv_off;
  double* ainv;
  const double* ebuf;
  const double* rbuf;
  const int64_t* bf_off;
  double* rnext;
  const double* ebuf2;
  const double* rbuf2;
  int rt_fixed, ct_fixed;
};

template <bool PAIR>
__global__ void __launch_bounds__(BF_THREADS, 3) k_bf_update(BfUpdArgs a) {
  extern __shared__ __align__(16) double bf_sm[];
  double(*Et)[BF_LDS] = reinterpret_cast<double(*)[BF_LDS]>(bf_sm);                 // [k][row]
  double(*Rt)[BF_LDS] = reinterpret_cast<double(*)[BF_LDS]>(bf_sm + BF_NB * BF_LDS);  // [col][k]
  __shared__ int s_oi;
  if (threadIdx.x < 32) {
    const int oi_w = bf_find_warp(a.pre, a.cnt, blockIdx.x);
    if (threadIdx.x == 0) s_oi = oi_w;
  }
  __syncthreads();
  const int L = a.L, j0 = a.j0;
  const int oi = s_oi;
  const int m = a.m_first + oi;
  const int n = L - m, lde = bf_lde(n);
  const int nt = (n + BF_T - 1) / BF_T;
  const int local = blockIdx.x - __ldg(a.pre + oi);
  const int jt = j0 / BF_T;
  int rt, ct;
  if (a.ct_fixed >= 0) {
    rt = local;
    ct = a.ct_fixed;
  } else if (a.rt_fixed >= 0) {
    rt = a.rt_fixed;
    ct = local;
    if (ct >= jt) ct += 2;  // skip J1 and J2
  } else {
    rt = local % nt;
    ct = local / nt;
    if (ct >= jt) ct += PAIR ? 2 : 1;  // skip the panel's column tile(s)
  }
  const int i0 = rt * BF_T, c0 = ct * BF_T;
  double* A = a.ainv + __ldg(a.ainv_off + m);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = (warp & 1) * 32, wc = (warp >> 1) * 16;  // warp tile 32 rows x 16 cols
  double acc[4][2][2];
#pragma unroll
  for (int h = 0; h < (PAIR ? 2 : 1); ++h) {
    const double* E = (h ? a.ebuf2 : a.ebuf) + __ldg(a.bf_off + m);
    const double* R = (h ? a.rbuf2 : a.rbuf) + __ldg(a.bf_off + m);
    const int nb = min(BF_NB, n - j0 - h * BF_NB);
    const int mlo = PAIR && h == 0 ? j0 + BF_NB : 0, mhi = PAIR && h == 0 ? j0 + 2 * BF_NB : 0;
    if (h) __syncthreads();  // the first half's operands are consumed
    // async staging: 64 x 64 doubles each = 2048 16-byte chunks, 8 per thread per operand
    for (int idx = tid; idx < BF_T * BF_NB / 2; idx += BF_THREADS) {
      const int k = idx >> 5, r2 = (idx & 31) * 2;  // E: column k, rows r2, r2+1
      const int row = i0 + r2;
      if (k < nb && row + 1 < lde && !(row >= mlo && row < mhi)) bf_cp16(&Et[k][r2], E + (int64_t)k * lde + row);
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
    if (h == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int row = i0 + wr + 8 * i + g, col = c0 + wc + 8 * j + 2 * t;
          acc[i][j][0] = (row < n && col < n) ? __ldcg(A + (int64_t)col * n + row) : 0.0;
          acc[i][j][1] = (row < n && col + 1 < n) ? __ldcg(A + (int64_t)(col + 1) * n + row) : 0.0;
        }
    }
    bf_cp_wait_all();
    __syncthreads();
#pragma unroll 4
    for (int k0 = 0; k0 < BF_NB; k0 += 4) {
      double av[4], bv[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = Et[k0 + t][wr + 8 * i + g];
#pragma unroll
      for (int j = 0; j < 2; ++j) bv[j] = Rt[wc + 8 * j + g][k0 + t];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
  }
  double* Rn = a.rnext ? a.rnext + __ldg(a.bf_off + m) : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int row = i0 + wr + 8 * i + g, col = c0 + wc + 8 * j + 2 * t;
      if (row < n && col < n) A[(int64_t)col * n + row] = acc[i][j][0];
      if (row < n && col + 1 < n) A[(int64_t)(col + 1) * n + row] = acc[i][j][1];
      if (Rn && i0 == j0 + BF_T && row < n) {  // the next panel's R = A[J', :] from the J' row tile
        if (col < n) Rn[(int64_t)col * BF_NB + (row - i0)] = acc[i][j][0];
        if (col + 1 < n) Rn[(int64_t)(col + 1) * BF_NB + (row - i0)] = acc[i][j][1];
      }
    }
}

// ---- 2c (wide). The same update on 128 x 64 tiles: eight warps of 32 x 32,
// so each k-step loads 8 fragments for 16 DMMAs (the 64 x 64 tile: 6 for 8)
// and every E / R element staged in shared memory feeds twice the math.
// 101 KB of shared memory, two CTAs per SM.  Default for L >= 1024
// (OSPH_BF_UPD_ROWS=64|128 forces either kernel).  Normal and PAIR modes.
#define BF_TW 128
#define BF_LDW (BF_TW + 4)
template <bool PAIR>
__global__ void __launch_bounds__(BF_THREADS, 2) k_bf_update_w(BfUpdArgs a) {
  extern __shared__ __align__(16) double bf_sm[];
  double(*Et)[BF_LDW] = reinterpret_cast<double(*)[BF_LDW]>(bf_sm);                  // [k][row]
  double(*Rt)[BF_LDS] = reinterpret_cast<double(*)[BF_LDS]>(bf_sm + BF_NB * BF_LDW);  // [col][k]
  __shared__ int s_oi;
  if (threadIdx.x < 32) {
    const int oi_w = bf_find_warp(a.pre, a.cnt, blockIdx.x);
    if (threadIdx.x == 0) s_oi = oi_w;
  }
  __syncthreads();
  const int L = a.L, j0 = a.j0;
  const int oi = s_oi;
  const int m = a.m_first + oi;
  const int n = L - m, lde = bf_lde(n);
  const int nt = (n + BF_TW - 1) / BF_TW;
  const int local = blockIdx.x - __ldg(a.pre + oi);
  const int rt = local % nt;
  int ct = local / nt;
  if (ct >= j0 / BF_T) ct += PAIR ? 2 : 1;  // skip the panel's column tile(s)
  const int i0 = rt * BF_TW, c0 = ct * BF_T;
  double* A = a.ainv + __ldg(a.ainv_off + m);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = (warp & 3) * 32, wc = (warp >> 2) * 32;  // warp tile 32 rows x 32 cols
  double acc[4][4][2];
#pragma unroll
  for (int h = 0; h < (PAIR ? 2 : 1); ++h) {
    const double* E = (h ? a.ebuf2 : a.ebuf) + __ldg(a.bf_off + m);
    const double* R = (h ? a.rbuf2 : a.rbuf) + __ldg(a.bf_off + m);
    const int nb = min(BF_NB, n - j0 - h * BF_NB);
    const int mlo = PAIR && h == 0 ? j0 + BF_NB : 0, mhi = PAIR && h == 0 ? j0 + 2 * BF_NB : 0;
    if (h) __syncthreads();
    for (int idx = tid; idx < BF_TW * BF_NB / 2; idx += BF_THREADS) {
      const int k = idx >> 6, r2 = (idx & 63) * 2;  // E: column k, rows r2, r2+1
      const int row = i0 + r2;
      if (k < nb && row + 1 < lde && !(row >= mlo && row < mhi)) bf_cp16(&Et[k][r2], E + (int64_t)k * lde + row);
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
    if (h == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int row = i0 + wr + 8 * i + g, col = c0 + wc + 8 * j + 2 * t;
          acc[i][j][0] = (row < n && col < n) ? __ldcg(A + (int64_t)col * n + row) : 0.0;
          acc[i][j][1] = (row < n && col + 1 < n) ? __ldcg(A + (int64_t)(col + 1) * n + row) : 0.0;
        }
    }
    bf_cp_wait_all();
    __syncthreads();
#pragma unroll 2
    for (int k0 = 0; k0 < BF_NB; k0 += 4) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = Et[k0 + t][wr + 8 * i + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Rt[wc + 8 * j + g][k0 + t];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
  }
  double* Rn = a.rnext ? a.rnext + __ldg(a.bf_off + m) : nullptr;
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

// ---- 4. coupling rows of the blocked sweep (sweep_block.cu):
//   U_m[r, j] = Pb_m[m-1-r, :] . X_m[:, j],   r < min(sb_rows(m), m),  j < n  (natural ring order),
// the response of ring m-1-r (a ring just below the block of order m) to entry j of order
// m's right-hand side.  Thread = column j (its 8-row pieces of the tiled X are contiguous;
// column 0, zeroed in the tiles, is w_m); the Pb rows are staged in shared memory and
// broadcast.  Output tiled like X (8-row tiles, 32-column chunks).
template <int J>
__device__ __forceinline__ void bf_couple_rows(int L, int m, const double* __restrict__ Xt,
                                               const double* __restrict__ Pb, const double* __restrict__ w,
                                               double* __restrict__ Ut, double* pbs) {
  // 128 threads = 32 columns x 4 row quarters: thread (column, quarter h) sums the 8-row
  // pieces it = h, h + 4, ... of its column (next piece prefetched); the quarters are added
  // in a fixed order by shuffles.
  const int n = L - m, nrt = (n + 7) >> 3, nrtpb = (m + 7) >> 3;
  const int JJ = min(J, m);
  const int cl = threadIdx.x >> 2, h = threadIdx.x & 3;
  const int cn = blockIdx.x * 32 + cl;
  const bool colok = cn < n;
  double acc[J];
#pragma unroll
  for (int r = 0; r < J; ++r) acc[r] = 0.0;
  const double* xcol = Xt + ((int64_t)(cn >> 5) * nrt << 8) + ((cn & 31) << 3);
  auto fetch = [&](int it, double (&x)[8]) {  // rows 8 it .. 8 it + 7 of column cn
    if (!colok || it >= nrt) {
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = 0.0;
    } else if (cn == 0) {  // the late ring's column is zero in the tiles: it is w_m (not padded)
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = (8 * it + q < n) ? __ldcg(w + 8 * it + q) : 0.0;
    } else {  // rows past n are zero in the tiles
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(xcol + (int64_t)it * 256 + q));
        x[q] = v.x;
        x[q + 1] = v.y;
      }
    }
  };
  for (int i0 = 0; i0 < n; i0 += 128) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < 128 * J; idx += 128) {  // pbs[i][r] = Pb[m-1-r, i0 + i]
      const int r = idx % J, i = idx / J;
      // two doubles of padding per 8-row piece: the four quarters of a warp read different banks
      pbs[idx + 2 * (i >> 3)] = (r < JJ && i0 + i < n) ? __ldcg(Pb + tile_index(m - 1 - r, i0 + i, nrtpb)) : 0.0;
    }
    __syncthreads();
    double xn[8];
    fetch((i0 >> 3) + h, xn);
#pragma unroll 1
    for (int t = h; t < 16; t += 4) {  // 16 pieces of 8 rows per 128-row chunk
      double x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = xn[q];
      fetch((i0 >> 3) + t + 4, xn);  // the first piece of the next chunk is fetched again there
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double* pr = pbs + (8 * t + q) * J + 2 * t;
#pragma unroll
        for (int r = 0; r < J; r += 2) {
          const double2 pv = *reinterpret_cast<const double2*>(pr + r);
          acc[r] = fma(pv.x, x[q], acc[r]);
          acc[r + 1] = fma(pv.y, x[q], acc[r + 1]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < J; ++r) {  // quarters 0 + 1 + 2 + 3, the same order on every lane
    const double a1 = __shfl_xor_sync(0xffffffffu, acc[r], 1);
    const double s01 = (h & 1) ? a1 + acc[r] : acc[r] + a1;
    const double a2 = __shfl_xor_sync(0xffffffffu, s01, 2);
    acc[r] = (h & 2) ? a2 + s01 : s01 + a2;
  }
  if (colok && h == 0) {
    double* out = Ut + (((int64_t)(cn >> 5) * (J / 8)) << 8) + ((cn & 31) << 3);
#pragma unroll
    for (int r = 0; r < J; ++r)
      if (r < JJ) out[(r >> 3) * 256 + (r & 7)] = acc[r];
  }
}

__global__ void __launch_bounds__(128) k_bf_couple(int L, int m_first, const int64_t* __restrict__ xt_off,
                                                   const double* __restrict__ xt_all,
                                                   const int64_t* __restrict__ pb_off,
                                                   const double* __restrict__ pbelow, const double* __restrict__ w_all,
                                                   const int64_t* __restrict__ ut_off, double* __restrict__ ut_all) {
  __shared__ __align__(16) double pbs[128 * OSPH_SB_BLOCK + 32];
  const int m = m_first + blockIdx.y;
  if (m == 0 || (int)blockIdx.x * 32 >= L - m) return;
  const double* Xt = xt_all + __ldg(xt_off + m);
  const double* Pb = pbelow + __ldg(pb_off + m);
  const double* w = w_all + (size_t)m * uw_ld(L);
  double* Ut = ut_all + __ldg(ut_off + m);
  if (m < OSPH_SB_BLOCK) bf_couple_rows<OSPH_SB_BLOCK>(L, m, Xt, Pb, w, Ut, pbs);
  else bf_couple_rows<OSPH_SB_BLOCK / 2>(L, m, Xt, Pb, w, Ut, pbs);
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
  // paired steps (rank-128 trailing updates)
  const int npsteps = (nmax + 2 * BF_NB - 1) / (2 * BF_NB);
  r->psteps.assign(npsteps, {});
  auto prefix = [&](int o0, int o1, auto items) {  // prefix table of orders m_first+o0 .. m_first+o1-1
    const int at = (int)tab.size();
    int acc = 0;
    for (int o = o0; o <= o1; ++o) {
      tab.push_back(acc);
      if (o < o1) acc += items(L - (m_first + o));
    }
    return std::make_pair(at, acc);
  };
  auto tiles = [](int n, int t) { return (n + t - 1) / t; };
  for (int ps = 0; ps < npsteps; ++ps) {
    auto& d = r->psteps[ps];
    d.j0 = ps * 2 * BF_NB;
    for (int m = m_first; m <= m_last; ++m) {
      if (L - m > d.j0) d.cnt = m - m_first + 1;
      if (L - m > d.j0 + BF_NB) d.cnt2 = m - m_first + 1;
    }
    std::tie(d.pre_panel, d.n_panel) = prefix(0, d.cnt, [&](int n) { return tiles(n, BF_T); });
    d.n_panel2 = tab[d.pre_panel + d.cnt2];
    std::tie(d.pre_row, d.n_row) = prefix(0, d.cnt2, [&](int n) { return tiles(n, BF_T) - 2; });
    std::tie(d.pre_upd2, d.n_upd2) = prefix(0, d.cnt2, [&](int n) { return tiles(n, BF_T) * (tiles(n, BF_T) - 2); });
    std::tie(d.pre_updw2, d.n_updw2) =
        prefix(0, d.cnt2, [&](int n) { return tiles(n, BF_TW) * (tiles(n, BF_T) - 2); });
    std::tie(d.pre_single, d.n_single) =
        prefix(d.cnt2, d.cnt, [&](int n) { return tiles(n, BF_T) * (tiles(n, BF_T) - 1); });
    std::tie(d.pre_singlew, d.n_singlew) =
        prefix(d.cnt2, d.cnt, [&](int n) { return tiles(n, BF_TW) * (tiles(n, BF_T) - 1); });
  }
  cudaError_t e;
  cudaFree(r->d_tab);
  r->d_tab = nullptr;
  if ((e = cudaMalloc(&r->d_tab, sizeof(int) * tab.size())) != cudaSuccess) return e;
  return cudaMemcpy(r->d_tab, tab.data(), sizeof(int) * tab.size(), cudaMemcpyHostToDevice);
}

static cudaError_t bf_attrs(int device) {
  static bool done[64] = {};  // per device (function attributes are per context)
  if (device >= 0 && device < 64 && done[device]) return cudaSuccess;
  const size_t sm2 = sizeof(double) * 2 * BF_T * BF_LDS + 16;
  const size_t smw = sizeof(double) * (BF_NB * BF_LDW + BF_T * BF_LDS) + 16;
  cudaError_t e = cudaFuncSetAttribute(k_bf_panel_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_bf_update<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_bf_update<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_bf_update_w<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_bf_update_w<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw);
  if (e == cudaSuccess && device >= 0 && device < 64) done[device] = true;
  return e;
}

// The blocks of orders r.m_first..r.m_last, rows in the order p->d_piv gives
// (plus, with the refinement buffer, the blocks in natural ring order).
cudaError_t bf_generate(osph_plan* p, const BfRange& r, cudaStream_t st, const BfOffsets& o, bool with_at) {
  const int L = p->L;
  const int cnt_all = r.m_last - r.m_first + 1;
  k_bf_generate<<<dim3((L + BF_THREADS - 1) / BF_THREADS, cnt_all), BF_THREADS, 0, st>>>(
      L, r.m_first, p->d_cos, p->d_rec, p->d_ls, p->d_pstart, p->d_piv, o.ainv, o.pb, p->d_ainv, p->d_pbelow);
  p->launches++;
  if (with_at && p->d_at) {  // the blocks themselves for the sweep's refinement step, natural ring order
    k_bf_generate_at<<<dim3((L + BF_THREADS - 1) / BF_THREADS, cnt_all), BF_THREADS, 0, st>>>(
        L, r.m_first, p->d_cos, p->d_rec, p->d_ls, p->d_pstart, o.xt, p->d_at);
    p->launches++;
  }
  return cudaGetLastError();
}

// One panel step (column block J = [j0, j0 + 64)) of every order with n > j0:
// R = A[J, :] (copied, or handed off by the previous step when fused_r),
// D = A[J, J]^{-1}, the panel E and the rank-64 update.
cudaError_t bf_step(osph_plan* p, const BfRange& r, int sidx, cudaStream_t st, const BfOffsets& o, bool fused_r) {
  const int L = p->L;
  const int m_first = r.m_first;
  cudaError_t e;
  if ((e = bf_attrs(p->device)) != cudaSuccess) return e;
  const size_t sm2 = sizeof(double) * 2 * BF_T * BF_LDS + 16;
  const size_t smw = sizeof(double) * (BF_NB * BF_LDW + BF_T * BF_LDS) + 16;
  // 128-row tiles win at large L (config 4: 1.574 vs 1.564 transforms/s), 64-row ones at L = 256
  // (config 2: 32.5k vs 32.3k); OSPH_BF_UPD_ROWS=64|128 forces one
  static const int upd_rows_env = getenv("OSPH_BF_UPD_ROWS") ? atoi(getenv("OSPH_BF_UPD_ROWS")) : 0;
  const bool upd_wide = upd_rows_env ? upd_rows_env == 128 : L >= 1024;
  const auto& d = r.steps[sidx];
  const int j0 = sidx * BF_NB;
  const dim3 dgrid(d.cnt, (L - m_first + BF_RCHUNK - 1) / BF_RCHUNK);
  double* rcur = p->d_bf_r + (fused_r ? (int64_t)(sidx & 1) * p->bf_r_half : 0);
  double* rnext = fused_r ? p->d_bf_r + (int64_t)((sidx + 1) & 1) * p->bf_r_half : nullptr;
  if (sidx == 0 || !fused_r) {
    k_bf_rcopy<<<dgrid, BF_THREADS, 0, st>>>(L, m_first, j0, o.ainv, p->d_ainv, rcur, o.bf);
    p->launches++;
  }
  k_bf_diag_rows<<<d.cnt, 64, 0, st>>>(L, m_first, j0, o.ainv, p->d_ainv, (r.dbuf ? r.dbuf : p->d_bf_d), p->d_status);
  k_bf_panel_mma<<<d.n_panel, BF_THREADS, sm2, st>>>(L, m_first, j0, r.d_tab + d.pre_panel, d.cnt, o.ainv,
                                                     p->d_ainv, (r.dbuf ? r.dbuf : p->d_bf_d), p->d_bf_e, o.bf, rnext);
  p->launches += 2;
  BfUpdArgs ua{L, m_first, j0, nullptr, d.cnt, o.ainv, p->d_ainv, p->d_bf_e, rcur, o.bf, rnext, nullptr, nullptr,
               -1, -1};
  if (d.n_upd > 0 && upd_wide) {
    ua.pre = r.d_tab + d.pre_updw;
    k_bf_update_w<false><<<d.n_updw, BF_THREADS, smw, st>>>(ua);
  } else if (d.n_upd > 0) {
    ua.pre = r.d_tab + d.pre_upd;
    k_bf_update<false><<<d.n_upd, BF_THREADS, sm2, st>>>(ua);
  }
  if (d.n_upd > 0) p->launches++;
  return cudaGetLastError();
}

// One paired step: the panels J1 = [j0, j0+64) and J2 = [j0+64, j0+128) of every
// order with n > j0 (J2 only where n > j0 + 64), with ONE pass of the trailing
// update over the matrix for both (rank 128) instead of two:
//   1  R1 = A[J1, :]                          6  D2 = A[J2, J2]^-1
//   2  D1 = A[J1, J1]^-1                      7  E2 = -A[:, J2] D2;  A[:, J2] = E2 + I
//   3  E1 = -A[:, J1] D1;  A[:, J1] = E1 + I  8  A[:, J1] += E2 R2[:, J1]
//      (and R2[:, J1] = A[J2, J1])            9  A[:, K] += E1' R1[:, K] + E2 R2[:, K]
//   4  A[:, J2] += E1 R1[:, J2]                  (K = outside J1, J2; E1' = E1 without the J2
//   5  A[J2, K] += E1[J2] R1[:, K];              rows, which step 5 already applied)
//      R2[:, K] = A[J2, K]
// Steps 4, 5 and 8 are 64-wide; step 9 is the bulk (2 n^2 128 flops per order).
// Orders whose n ends inside J2's range take the rank-64 update of J1 instead.
static cudaError_t bf_pair_step(osph_plan* p, const BfRange& r, int ps, cudaStream_t st, const BfOffsets& o,
                                bool upd_wide) {
  const int L = p->L;
  const int m_first = r.m_first;
  const BfPairStep& d = r.psteps[ps];
  const int j0 = d.j0, jt = j0 / BF_T;
  const size_t sm2 = sizeof(double) * 2 * BF_T * BF_LDS + 16;
  const size_t smw = sizeof(double) * (BF_NB * BF_LDW + BF_T * BF_LDS) + 16;
  double* R1 = p->d_bf_r;
  double* R2 = p->d_bf_r + p->bf_r_half;
  const int* tab = r.d_tab;
  const dim3 dgrid(d.cnt, (L - m_first + BF_RCHUNK - 1) / BF_RCHUNK);
  k_bf_rcopy<<<dgrid, BF_THREADS, 0, st>>>(L, m_first, j0, o.ainv, p->d_ainv, R1, o.bf);                // 1
  k_bf_diag_rows<<<d.cnt, 64, 0, st>>>(L, m_first, j0, o.ainv, p->d_ainv, (r.dbuf ? r.dbuf : p->d_bf_d), p->d_status);     // 2
  k_bf_panel_mma<<<d.n_panel, BF_THREADS, sm2, st>>>(L, m_first, j0, tab + d.pre_panel, d.cnt, o.ainv,  // 3
                                                     p->d_ainv, (r.dbuf ? r.dbuf : p->d_bf_d), p->d_bf_e, o.bf, d.cnt2 ? R2 : nullptr);
  p->launches += 3;
  if (d.cnt2 > 0) {
    BfUpdArgs u{L, m_first, j0, tab + d.pre_panel, d.cnt2, o.ainv, p->d_ainv, p->d_bf_e, R1, o.bf, nullptr,
                nullptr, nullptr, -1, jt + 1};
    k_bf_update<false><<<d.n_panel2, BF_THREADS, sm2, st>>>(u);  // 4
    u.pre = tab + d.pre_row;
    u.ct_fixed = -1;
    u.rt_fixed = jt + 1;
    u.rnext = R2;
    if (d.n_row > 0) k_bf_update<false><<<d.n_row, BF_THREADS, sm2, st>>>(u);  // 5
    k_bf_diag_rows<<<d.cnt2, 64, 0, st>>>(L, m_first, j0 + BF_NB, o.ainv, p->d_ainv, (r.dbuf ? r.dbuf : p->d_bf_d), p->d_status);  // 6
    k_bf_panel_mma<<<d.n_panel2, BF_THREADS, sm2, st>>>(L, m_first, j0 + BF_NB, tab + d.pre_panel, d.cnt2,     // 7
                                                        o.ainv, p->d_ainv, (r.dbuf ? r.dbuf : p->d_bf_d), p->d_bf_e2, o.bf, nullptr);
    BfUpdArgs v{L, m_first, j0 + BF_NB, tab + d.pre_panel, d.cnt2, o.ainv, p->d_ainv, p->d_bf_e2, R2, o.bf,
                nullptr, nullptr, nullptr, -1, jt};
    k_bf_update<false><<<d.n_panel2, BF_THREADS, sm2, st>>>(v);  // 8
    BfUpdArgs w{L, m_first, j0, nullptr, d.cnt2, o.ainv, p->d_ainv, p->d_bf_e, R1, o.bf, nullptr, p->d_bf_e2, R2,
                -1, -1};
    if (upd_wide && d.n_updw2 > 0) {  // 9
      w.pre = tab + d.pre_updw2;
      k_bf_update_w<true><<<d.n_updw2, BF_THREADS, smw, st>>>(w);
    } else if (d.n_upd2 > 0) {
      w.pre = tab + d.pre_upd2;
      k_bf_update<true><<<d.n_upd2, BF_THREADS, sm2, st>>>(w);
    }
    p->launches += 6;
  }
  if (d.cnt > d.cnt2) {  // orders without a J2 panel in this step: the rank-64 update of J1
    BfUpdArgs u{L, m_first + d.cnt2, j0, nullptr, d.cnt - d.cnt2, o.ainv, p->d_ainv, p->d_bf_e, R1, o.bf, nullptr,
                nullptr, nullptr, -1, -1};
    if (upd_wide && d.n_singlew > 0) {
      u.pre = tab + d.pre_singlew;
      k_bf_update_w<false><<<d.n_singlew, BF_THREADS, smw, st>>>(u);
      p->launches++;
    } else if (d.n_single > 0) {
      u.pre = tab + d.pre_single;
      k_bf_update<false><<<d.n_single, BF_THREADS, sm2, st>>>(u);
      p->launches++;
    }
  }
  return cudaGetLastError();
}

// Factor orders r.m_first..r.m_last with the recorded pivot order, writing A/X,
// Pb, the tiled X and the sweep constants at the given offset tables.
cudaError_t bf_run(osph_plan* p, const BfRange& r, cudaStream_t st, const BfOffsets& o) {
  const int L = p->L;
  const int m_first = r.m_first;
  const int cnt_all = r.m_last - r.m_first + 1;
  cudaError_t e;
  if ((e = bf_generate(p, r, st, o, true)) != cudaSuccess) return e;
  if (p->need_norms) {  // ||A||_1 and ||X||_1 feed only the check=True condition estimate
    k_bf_colnorm<<<dim3(8, cnt_all), BF_THREADS, 0, st>>>(L, m_first, o.ainv, p->d_ainv, p->d_norms, 0);
    p->launches++;
  }
  // R = A[J, :] of a step: copied at step 0; afterwards written by the previous
  // step's panel (J columns) and update (J-row tiles) into the other of two
  // buffers (OSPH_BF_RFUSE=0 copies it every step instead; bit-identical)
  static const bool fused_r = !(getenv("OSPH_BF_RFUSE") && atoi(getenv("OSPH_BF_RFUSE")) == 0);
  // paired (rank-128) steps: half the passes of the trailing update over every matrix
  // (measured: config 4 1.755 vs 1.567 transforms/s, config 2 33.5k vs 33.2k);
  // OSPH_BF_PAIR=0 forces the rank-64 steps
  static const int pair_env = getenv("OSPH_BF_PAIR") ? atoi(getenv("OSPH_BF_PAIR")) : -1;
  const bool paired = pair_env != 0;
  if (paired) {
    if ((e = bf_attrs(p->device)) != cudaSuccess) return e;
    static const int upd_rows_env = getenv("OSPH_BF_UPD_ROWS") ? atoi(getenv("OSPH_BF_UPD_ROWS")) : 0;
    const bool upd_wide = upd_rows_env ? upd_rows_env == 128 : L >= 1024;
    for (size_t ps = 0; ps < r.psteps.size(); ++ps)
      if ((e = bf_pair_step(p, r, (int)ps, st, o, upd_wide)) != cudaSuccess) return e;
  } else {
    for (size_t sidx = 0; sidx < r.steps.size(); ++sidx)
      if ((e = bf_step(p, r, (int)sidx, st, o, fused_r)) != cudaSuccess) return e;
  }
  if (p->need_norms) {
    k_bf_colnorm<<<dim3(8, cnt_all), BF_THREADS, 0, st>>>(L, m_first, o.ainv, p->d_ainv, p->d_norms, 1);
    p->launches++;
  }
  k_bf_epilogue<<<dim3(8, cnt_all), BF_THREADS, 0, st>>>(L, m_first, o.ainv, p->d_ainv, p->d_piv, o.xt, p->d_xt,
                                                         o.pb, p->d_pbelow, p->d_u, p->d_w, p->d_beta, p->d_jstar);
  p->launches++;
  if (p->d_ut && !p->windowed && L <= 1024) {  // resident plans: the coupling rows of the blocked sweep
    k_bf_couple<<<dim3((L - m_first + 31) / 32, cnt_all), 128, 0, st>>>(L, m_first, o.xt, p->d_xt, o.pb, p->d_pbelow,
                                                                       p->d_w, p->d_ut_off, p->d_ut);
    p->launches++;
  }
  return cudaGetLastError();
}

// The non-windowed plan: orders m_first..m_last, full offset tables.
cudaError_t launch_factor_bf(osph_plan* p, int m_first, int m_last, cudaStream_t st) {
  cudaError_t e;
  if (p->bf_full.m_first != m_first || p->bf_full.m_last != m_last)
    if ((e = bf_prepare(p, m_first, m_last, &p->bf_full)) != cudaSuccess) return e;
  const BfOffsets o{p->d_ainv_off, p->d_xt_off, p->d_pb_off, p->d_bf_off};
  return bf_run(p, p->bf_full, st, o);
}
