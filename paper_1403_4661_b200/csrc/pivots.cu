// pivots.cu -- the grid's pivot order for every per-order block (once per grid).
//
// The per-order blocks A_m = 2pi Y_lm(theta_k) (rings k >= m as rows, degrees
// l >= m as columns; transform.py:416-429) depend only on the grid, and so
// does the row order that partial pivoting picks for them.  The reference
// solves each block with LAPACK gelsy (QR with column pivoting,
// blocks.py:88-116); here the blocks are inverted by Gauss-Jordan with the
// row order of LU with partial pivoting (LU vs gelsy: max|df| 2.2e-14 at
// L=512), and that order is found by this file, in house:
//
//   the breadth-first factorisation of factor_bf.cu (rows in natural ring
//   order), with a partial-pivoting search in front of every 64-column panel
//   step.  For the columns J = [j0, j0 + 64) of every order the remaining
//   rows (positions >= j0) hold the Schur complement, so a tall-skinny LU with
//   partial pivoting of A[j0:, J] (k_piv_panel) picks exactly the 64 pivots
//   right-looking blocked LU with partial pivoting (LAPACK getrf) would pick
//   at those columns: largest |value| of the current column, first position on
//   ties (idamax), rows exchanged LAPACK-style.  k_piv_swap then moves those
//   rows into positions j0 .. j0 + 63 of the whole matrix (and of perm_m), and
//   the ordinary static-pivot step (bf_step) eliminates them.
//
// k_piv_panel keeps one row of the n_rem x 64 panel per thread in registers,
// rotated so the current column is register 0 (as k_bf_diag_rows), with up to
// 4096 rows on a cluster of up to 16 CTAs: per pivot, a CTA-local argmax, the
// CTA winner's row pushed into every CTA's shared memory (DSMEM stores), one
// cluster barrier, the same global winner chosen by every CTA, and the rank-1
// update of every row.  Result: perm_m[i] = ring offset at pivot position i
// in p->d_piv, cached per grid (process-wide) so later plans on the same grid
// only upload it.  No library factorisation is involved.
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <climits>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/osph.h"
#include "plan.cuh"

namespace cg = cooperative_groups;

#define PV_THREADS 256
#define PV_NB 64          // = BF_NB (factor_bf.cu)
#define PV_REC (PV_NB + 2)  // candidate record: columns p+1 .. p+63, signed pivot value, position
#define PV_MOVES 128      // at most 2 rows change position per pivot

template <int CS>
__global__ void __launch_bounds__(PV_THREADS, 1) k_piv_panel(int L, int m_lo, int j0,
                                                             const int64_t* __restrict__ ainv_off,
                                                             const double* __restrict__ ainv,
                                                             int* __restrict__ moves, int* __restrict__ nmoves) {
  __shared__ __align__(16) double s_stage[PV_REC];
  __shared__ __align__(16) double s_cand[2][CS][PV_REC];
  __shared__ double s_wv[PV_THREADS / 32];
  __shared__ int s_wp[PV_THREADS / 32], s_wt[PV_THREADS / 32];
  __shared__ int s_bt, s_bp;
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  const int m = m_lo + blockIdx.x / CS;
  const int n = L - m;
  const int nb = min(PV_NB, n - j0);
  const double* A = ainv + __ldg(ainv_off + m);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int pos0 = j0 + crank * PV_THREADS + t;
  const bool active = pos0 < n;
  int pos = pos0;
  bool done = !active;
  double d[PV_NB];
#pragma unroll
  for (int c = 0; c < PV_NB; ++c) d[c] = (active && c < nb) ? __ldcg(A + (int64_t)(j0 + c) * n + pos0) : 0.0;
#pragma unroll 1
  for (int p = 0; p < nb; ++p) {
    // ---- CTA-local argmax of |column p| over the rows not yet pivoted (ties: lowest position)
    double v = done ? -1.0 : fabs(d[0]);
    if (v != v) v = 0.0;  // NaN: eligible only when nothing else is (the diagonal inverse flags it)
    int bp = done ? INT_MAX : pos, bt = t;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
      if (ov > v || (ov == v && op < bp)) {
        v = ov;
        bp = op;
        bt = ot;
      }
    }
    if (lane == 0) {
      s_wv[warp] = v;
      s_wp[warp] = bp;
      s_wt[warp] = bt;
    }
    __syncthreads();
    if (warp == 0) {
      v = lane < PV_THREADS / 32 ? s_wv[lane] : -2.0;
      bp = lane < PV_THREADS / 32 ? s_wp[lane] : INT_MAX;
      bt = lane < PV_THREADS / 32 ? s_wt[lane] : 0;
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
        if (ov > v || (ov == v && op < bp)) {
          v = ov;
          bp = op;
          bt = ot;
        }
      }
      if (lane == 0) {
        s_bt = bt;
        s_bp = bp;
      }
    }
    __syncthreads();
    // ---- the CTA's candidate (its winner's remaining columns, value, position) -> every CTA
    if (s_bp == INT_MAX) {
      if (t == 0) {
        s_stage[PV_NB - 1] = 0.0;
        s_stage[PV_NB] = 1e300;  // no candidate in this CTA
      }
    } else if (t == s_bt) {
#pragma unroll
      for (int c = 0; c < PV_NB - 1; ++c) s_stage[c] = d[c + 1];
      s_stage[PV_NB - 1] = d[0];
      s_stage[PV_NB] = (double)pos;
    }
    __syncthreads();
    for (int i = t; i < CS * PV_REC; i += PV_THREADS) {
      const int r = i / PV_REC, c = i - r * PV_REC;
      double* dst = cl.map_shared_rank(&s_cand[p & 1][crank][0], r);
      dst[c] = s_stage[c];
    }
    cl.sync();
    // ---- the global winner (every CTA computes the same one)
    int w = 0;
    double wv = -1.0, wp = 1e300;
#pragma unroll
    for (int r = 0; r < CS; ++r) {
      double cv = fabs(s_cand[p & 1][r][PV_NB - 1]);
      if (cv != cv) cv = 0.0;
      const double cp = s_cand[p & 1][r][PV_NB];
      if (cp < 1e299 && (cv > wv || (cv == wv && cp < wp))) {
        w = r;
        wv = cv;
        wp = cp;
      }
    }
    const double* prow = s_cand[p & 1][w];
    const double pv = prow[PV_NB - 1];
    const int q = (int)prow[PV_NB];
    // LAPACK-style exchange of positions j0 + p and q
    if (!done && pos == q) {
      done = true;
      pos = j0 + p;
    } else if (pos == j0 + p) {
      pos = q;
    }
    const double g = (!done && pv != 0.0 && pv == pv) ? d[0] / pv : 0.0;
#pragma unroll
    for (int c = 0; c < PV_NB - 1; ++c) d[c] = fma(-g, prow[c], d[c + 1]);
    d[PV_NB - 1] = 0.0;
  }
  // rows whose position changed: (destination, source) pairs for k_piv_swap
  if (active && pos != pos0) {
    const int i = atomicAdd(nmoves + m, 1);
    if (i < PV_MOVES) {
      moves[((int64_t)m * PV_MOVES + i) * 2] = pos;
      moves[((int64_t)m * PV_MOVES + i) * 2 + 1] = pos0;
    }
  }
}

// Apply the panel's row moves to every column of A_m and to perm_m:
// new[dst] = old[src].  Grid (orders, column chunks); warp per column.
__global__ void __launch_bounds__(PV_THREADS) k_piv_swap(int L, int m_first, const int64_t* __restrict__ ainv_off,
                                                         double* __restrict__ ainv, const int* __restrict__ moves,
                                                         const int* __restrict__ nmoves, int* __restrict__ perm_all) {
  __shared__ int s_dst[PV_MOVES], s_src[PV_MOVES];
  const int m = m_first + blockIdx.x;
  const int n = L - m;
  const int cnt = min(__ldg(nmoves + m), PV_MOVES);
  if (cnt == 0) return;
  for (int i = threadIdx.x; i < cnt; i += PV_THREADS) {
    s_dst[i] = __ldg(moves + ((int64_t)m * PV_MOVES + i) * 2);
    s_src[i] = __ldg(moves + ((int64_t)m * PV_MOVES + i) * 2 + 1);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* A = ainv + __ldg(ainv_off + m);
  constexpr int PER = PV_MOVES / 32;
  for (int c = blockIdx.y * (PV_THREADS / 32) + warp; c <= n; c += gridDim.y * (PV_THREADS / 32)) {
    if (c == n) {  // the permutation itself (exactly one warp of the grid gets c == n)
      int* perm = perm_all + packed_pos(L, m, 0);
      int v[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) v[u] = (lane + 32 * u < cnt) ? perm[s_src[lane + 32 * u]] : 0;
      __syncwarp();
#pragma unroll
      for (int u = 0; u < PER; ++u)
        if (lane + 32 * u < cnt) perm[s_dst[lane + 32 * u]] = v[u];
      continue;
    }
    double* col = A + (int64_t)c * n;
    double v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) v[u] = (lane + 32 * u < cnt) ? __ldcg(col + s_src[lane + 32 * u]) : 0.0;
    __syncwarp();
#pragma unroll
    for (int u = 0; u < PER; ++u)
      if (lane + 32 * u < cnt) col[s_dst[lane + 32 * u]] = v[u];
  }
}

template <int CS>
static cudaError_t launch_piv_panel(osph_plan* p, int m_lo, int m_hi, int j0, const int64_t* ainv_off, int* moves,
                                    int* nmoves, cudaStream_t st) {
  auto kern = k_piv_panel<CS>;
  cudaError_t e;
  if (CS > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((m_hi - m_lo + 1) * CS));
  cfg.blockDim = dim3(PV_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  p->launches++;
  return cudaLaunchKernelEx(&cfg, kern, p->L, m_lo, j0, ainv_off, (const double*)p->d_ainv, moves, nmoves);
}

// Pivot search + row exchange of step sidx for the orders of range r, then the
// static-pivot step itself.  h_ainv_off: host copy of the range's A offsets.
static cudaError_t pivot_step(osph_plan* p, const BfRange& r, int sidx, const BfOffsets& o, int* moves, int* nmoves,
                              cudaStream_t st) {
  const int L = p->L;
  const int j0 = sidx * PV_NB;
  const int cnt = r.steps[sidx].cnt;  // orders m_first .. m_first + cnt - 1 have n > j0
  if (cnt == 0) return cudaSuccess;
  cudaError_t e;
  if ((e = cudaMemsetAsync(nmoves, 0, sizeof(int) * L, st)) != cudaSuccess) return e;
  // classes by remaining rows n - j0: cluster size = CTAs of 256 rows (1 .. 16)
  int m = r.m_first;
  const int m_end = r.m_first + cnt - 1;
  while (m <= m_end) {
    const int rows = L - m - j0;
    int cs = 1;
    while (cs * PV_THREADS < rows) cs *= 2;
    // orders m .. mb share this cluster size (rows decrease with m)
    int mb = m;
    while (mb + 1 <= m_end) {
      const int rr = L - (mb + 1) - j0;
      int c2 = 1;
      while (c2 * PV_THREADS < rr) c2 *= 2;
      if (c2 != cs) break;
      ++mb;
    }
    switch (cs) {
      case 1: e = launch_piv_panel<1>(p, m, mb, j0, o.ainv, moves, nmoves, st); break;
      case 2: e = launch_piv_panel<2>(p, m, mb, j0, o.ainv, moves, nmoves, st); break;
      case 4: e = launch_piv_panel<4>(p, m, mb, j0, o.ainv, moves, nmoves, st); break;
      case 8: e = launch_piv_panel<8>(p, m, mb, j0, o.ainv, moves, nmoves, st); break;
      default: e = launch_piv_panel<16>(p, m, mb, j0, o.ainv, moves, nmoves, st); break;
    }
    if (e != cudaSuccess) return e;
    m = mb + 1;
  }
  const int nmax = L - r.m_first;
  k_piv_swap<<<dim3(cnt, std::min(64, (nmax + 1 + 7) / 8)), PV_THREADS, 0, st>>>(L, r.m_first, o.ainv, p->d_ainv,
                                                                                moves, nmoves, p->d_piv);
  p->launches++;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return bf_step(p, r, sidx, st, o, false);
}

namespace {
std::mutex g_piv_mu;
std::map<std::vector<double>, std::vector<int>> g_piv_cache;  // thetas -> perm (packed by order)
}  // namespace

#define PIV_TRY(expr)                                                      \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess) {                                               \
      osph_set_error(std::string("pivot discovery: ") + #expr + ": " + cudaGetErrorString(_e)); \
      rc = OSPH_ERR_CUDA;                                                  \
      goto done;                                                           \
    }                                                                      \
  } while (0)

// Fills p->d_piv (perm[packed_pos(L, m, i)] = ring offset at pivot position i)
// and sets p->piv_ready.  Host-blocking; runs on the plan stream.  Needs the
// factor storage (ensure_forward) in place.
int discover_pivots(osph_plan* p) {
  const int L = p->L;
  const int64_t npk = (int64_t)L * (L + 1) / 2;
  cudaStream_t st = p->stream;
  int rc = OSPH_OK;
  int* moves = nullptr;
  int* nmoves = nullptr;
  std::vector<double> key(L);
  std::vector<int> perm(npk);
  {  // thetas of the plan (cos is stored; the key only has to identify the grid)
    if (cudaMemcpy(key.data(), p->d_cos, sizeof(double) * L, cudaMemcpyDeviceToHost) != cudaSuccess) {
      osph_set_error("pivot discovery: reading the grid");
      return OSPH_ERR_CUDA;
    }
    std::lock_guard<std::mutex> lk(g_piv_mu);
    auto it = g_piv_cache.find(key);
    if (it != g_piv_cache.end() && !getenv("OSPH_PIVOTS_NOCACHE")) {  // (tests: force a fresh discovery)
      if (cudaMemcpy(p->d_piv, it->second.data(), sizeof(int) * npk, cudaMemcpyHostToDevice) != cudaSuccess) {
        osph_set_error("pivot discovery: upload");
        return OSPH_ERR_CUDA;
      }
      p->piv_ready = true;
      return OSPH_OK;
    }
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (int m = 0; m < L; ++m)
    for (int i = 0; i < L - m; ++i) perm[packed_pos(L, m, i)] = i;
  PIV_TRY(cudaMemcpyAsync(p->d_piv, perm.data(), sizeof(int) * npk, cudaMemcpyHostToDevice, st));
  PIV_TRY(cudaMalloc(&moves, sizeof(int) * 2 * PV_MOVES * (size_t)L));
  PIV_TRY(cudaMalloc(&nmoves, sizeof(int) * (size_t)L));
  PIV_TRY(cudaMemsetAsync(p->d_status, 0, sizeof(int) * L, st));
  if (!p->windowed) {
    int lo, hi;
    own_orders(p, lo, hi);  // a factor shard needs (and finds) only its own orders' pivots
    if (p->bf_full.m_first != lo || p->bf_full.m_last != hi) PIV_TRY(bf_prepare(p, lo, hi, &p->bf_full));
    const BfOffsets o{p->d_ainv_off, p->d_xt_off, p->d_pb_off, p->d_bf_off};
    PIV_TRY(bf_generate(p, p->bf_full, st, o, false));
    for (size_t s = 0; s < p->bf_full.steps.size(); ++s)
      PIV_TRY(pivot_step(p, p->bf_full, (int)s, o, moves, nmoves, st));
  } else {
    for (FwdWindow& w : p->windows) {
      const BfOffsets o{w.d_offs, w.d_offs + (L + 1), w.d_offs + 2 * (L + 1), w.d_offs + 3 * (L + 1)};
      PIV_TRY(bf_generate(p, w.bf, st, o, false));
      for (size_t s = 0; s < w.bf.steps.size(); ++s) PIV_TRY(pivot_step(p, w.bf, (int)s, o, moves, nmoves, st));
    }
  }
  PIV_TRY(cudaMemcpyAsync(perm.data(), p->d_piv, sizeof(int) * npk, cudaMemcpyDeviceToHost, st));
  PIV_TRY(cudaMemsetAsync(p->d_status, 0, sizeof(int) * L, st));
  PIV_TRY(cudaStreamSynchronize(st));
  if (!p->shard_mode) {  // a shard's discovery covers only its orders: not a complete entry
    std::lock_guard<std::mutex> lk(g_piv_mu);
    if (g_piv_cache.size() >= 16) g_piv_cache.erase(g_piv_cache.begin());
    g_piv_cache[key] = perm;
  }
  p->piv_ready = true;
  p->pivot_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
done:
  cudaFree(moves);
  cudaFree(nmoves);
  return rc;
}
