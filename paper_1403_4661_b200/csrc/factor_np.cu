// factor_np.cu -- per-order inversion with STATIC pivots, shared-memory resident.
//
// The per-order blocks A_m = 2pi Y_lm(theta_k, 0) depend only on the grid, so
// the row order chosen by partial pivoting is the same on every call.  The
// first forward transform of a plan runs the pivoting kernel (factor.cu),
// which records perm_m (O(L^2) integers, kept in the plan next to the other
// O(L^2) tables -- the reference likewise caches O(L^2) tables per band
// limit, transform.py:268-301).  Every later call regenerates A_m in that row
// order and inverts it by blocked Gauss-Jordan WITHOUT a pivot search -- the
// identical elimination sequence -- which turns each panel step into an
// unblocked elimination of the n x 32 panel (one row per thread, in
// registers, one barrier per pivot) plus one GEMM on the fp64 tensor cores:
//     [E + I on P] = GJ(A[:, P]),  A[:, rest] += E A[P, rest].
// The O(L^3) work (generation + inversion) is still done per call.
//
// One thread-block cluster per order; CTA r owns a contiguous slice of the
// columns, held in shared memory for the whole factorisation (n <= 256), so
// row interchanges never happen and every update is smem-to-smem.  The panel
// owner publishes each panel through a small global buffer (double-buffered)
// and one cluster barrier per panel orders the hand-off.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <utility>

#include "plan.cuh"

namespace cg = cooperative_groups;

#define FNP_THREADS 256
#define FNP_WARPS 8
#define FNP_NB 32

#ifdef OSPH_FACTOR_PROF
#define FNP_MARK(i)                                   \
  do {                                                \
    if (threadIdx.x == 0) {                           \
      const long long _n = clock64();                 \
      _fa[i] += _n - _ft;                             \
      _ft = _n;                                       \
    }                                                 \
  } while (0)
#else
#define FNP_MARK(i)
#endif

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }

__device__ __forceinline__ void np_atomic_max_pos(unsigned long long* addr, double v) {
  if (!(v >= 0.0) || isinf(v)) v = INFINITY;
  atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

struct NpLayout {
  int ldn, cwmax;
  size_t slice, es, rowbuf, pinv_bytes_off, total_doubles;
  __host__ __device__ NpLayout(int nmax, int CS) {
    ldn = ((nmax + 15) / 16) * 16 + 4;
    const int units = (nmax + FNP_NB - 1) / FNP_NB;
    cwmax = ((units + CS - 1) / CS) * FNP_NB;
    size_t o = 0;
    slice = o;  o += (size_t)cwmax * ldn;
    es = o;     o += (size_t)FNP_NB * ldn;
    rowbuf = o; o += 2 * FNP_NB;
    pinv_bytes_off = o;  // ints follow
    o += (size_t)(nmax + 1) / 2 + 1;
    total_doubles = o;
  }
};

__global__ void __launch_bounds__(FNP_THREADS, 1) k_factor_np(
    int L, int m_first, int nmax, const double* __restrict__ costh, const double2* __restrict__ rec,
    const int* __restrict__ ls_tab, const double2* __restrict__ pstart, const int* __restrict__ perm_all,
    double* __restrict__ xt_all, const int64_t* __restrict__ xt_off, double* __restrict__ pbelow,
    const int64_t* __restrict__ pb_off, double* __restrict__ panel_g, unsigned long long* __restrict__ norms,
    int* __restrict__ status_out, int* __restrict__ jstar_out, double* __restrict__ beta_out,
    double* __restrict__ u_out, double* __restrict__ w_out) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int slot = (int)(blockIdx.x / CS);
  const int m = m_first + slot;
  if (m >= L) return;
  const int n = L - m;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;

  extern __shared__ __align__(16) double smem[];
  const NpLayout lay(nmax, CS);
  const int ldn = lay.ldn;
  double* slice = smem + lay.slice;    // own columns, column-major, ld = ldn
  double* Es = smem + lay.es;          // panel / E, column-major [NB][ldn]
  double* rowbuf = smem + lay.rowbuf;  // scaled pivot row broadcast, double-buffered
  int* pinv = reinterpret_cast<int*>(smem + lay.pinv_bytes_off);
  __shared__ int s_bad;
  __shared__ double s_red[FNP_WARPS];

  const int* perm = perm_all + packed_pos(L, m, 0);
  const int units = (n + FNP_NB - 1) / FNP_NB;
  const int u0 = (rank * units) / CS, u1 = ((rank + 1) * units) / CS;
  const int c0 = u0 * FNP_NB, c1 = min(n, u1 * FNP_NB);
  const int cw = max(0, c1 - c0);
  const int cwt = (cw + 7) & ~7;  // own columns rounded to 8-column tiles
  const int nrt8 = (n + 7) >> 3;
  // hand-off slot per order (classes may run concurrently on different streams)
  const int nall = min(L, 256), ldn_all = ((nall + 15) / 16) * 16 + 4;
  double* pg = panel_g + (size_t)(m - (L - nall)) * 2 * FNP_NB * ldn_all;

  if (tid == 0) s_bad = 0;
#ifdef OSPH_FACTOR_PROF
  long long _ft = clock64(), _fa[6] = {0, 0, 0, 0, 0, 0};
#endif
  for (int j = tid; j < n; j += FNP_THREADS) pinv[__ldg(perm + j)] = j;
  // Rows n..ldn-1 of the slice and of Es are read by the 8-row tiles and the
  // k-steps of the last panel (multiplied by zero E entries): they must hold
  // zeros, not whatever the previous kernel left in shared memory (Es follows
  // the slice, so the columns of both are one range).  Own padding columns
  // cw..cwt-1 are zeroed whole.
  for (int c = warp; c < lay.cwmax + FNP_NB; c += FNP_WARPS)
    for (int r = (c >= cw && c < lay.cwmax ? 0 : n) + lane; r < ldn; r += 32) slice[(size_t)c * ldn + r] = 0.0;

  // ---- 1. generation: own degree columns l = m+c0 .. m+c1-1, rows in pivot order;
  //         rings k < m go to the tiled below-block Pb (sweep operand)
  {
    const double2* recm = rec + packed_pos(L, m, 0);
    double* Pb = pbelow + pb_off[m];
    const int nrtpb = (m + 7) >> 3;
    for (int it = tid; it < L; it += FNP_THREADS) {
      const int k = it < n ? m + __ldg(perm + it) : it - n;  // row item -> ring
      const int64_t t = (int64_t)m * L + k;
      const int ls = ls_tab[t];
      const double2 pp = pstart[t];
      double p0 = pp.x, p1 = pp.y;
      const double x = costh[k];
      for (int l = m; l < m + c1; ++l) {
        double v = 0.0;
        if (l >= ls) {
          v = OSPH_TWO_PI * p1;
          const double2 ar = __ldg(recm + (l - m));
          const double nxt = fma(x, p1, -ar.x * p0) * ar.y;
          p0 = p1;
          p1 = nxt;
        }
        if (l >= m + c0) {
          if (it < n) slice[(size_t)(l - m - c0) * ldn + it] = v;
          else Pb[tile_index(k, l - m, nrtpb)] = v;
        }
      }
    }
  }
  __syncthreads();
  // ||A||_1 over own columns
  {
    double cmax = 0.0;
    for (int c = warp; c < cw; c += FNP_WARPS) {
      double s = 0.0;
      for (int i = lane; i < n; i += 32) s += fabs(slice[(size_t)c * ldn + i]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      cmax = fmax(cmax, s);
    }
    if (lane == 0 && cw > 0) np_atomic_max_pos(norms + 2 * m, cmax);
  }

  FNP_MARK(0);
  // ---- 2. blocked Gauss-Jordan, static pivots
  const int nct = cwt >> 3;  // own 8-column tiles
  auto export_panel = [&](int jp, double* dst) {  // own columns jp .. jp+nb-1 -> global
    const int nbp = min(FNP_NB, n - jp);
    for (int c = warp; c < nbp; c += FNP_WARPS)
      for (int r = lane; r < n; r += 32) dst[(size_t)c * ldn + r] = slice[(size_t)(jp - c0 + c) * ldn + r];
  };
  for (int j0 = 0, par = 0; j0 < n; j0 += FNP_NB, par ^= 1) {
    const int nb = min(FNP_NB, n - j0);
    const bool owner = j0 >= c0 && j0 < c1;
    double* pgp = pg + (size_t)par * FNP_NB * ldn;
    if (owner) export_panel(j0, pgp);
    cluster_arrive();
    cluster_wait();
    FNP_MARK(1);
    // a) panel -> registers, thread = row (columns >= nb zero)
    double d[FNP_NB];
    const bool hasrow = tid < n;
#pragma unroll
    for (int c = 0; c < FNP_NB; ++c)
      d[c] = (hasrow && c < nb) ? __ldcg(pgp + (size_t)c * ldn + tid) : 0.0;
    FNP_MARK(2);
    // b) unblocked Gauss-Jordan on the n x nb panel (the same elimination the
    //    full in-place inversion applies to these columns), one row per thread
    //    in registers.  The row is kept ROTATED so that the current pivot column
    //    is always d[0]: step p maps d[c] <- column (p + c) mod 32, so the loop
    //    body has static register indices and stays rolled (the code runs 32
    //    times per panel from the instruction cache).  Pivot row r = j0 + p is
    //    published unscaled with its reciprocal (double-buffered: one barrier
    //    per pivot); every other row subtracts g = f / piv times it, and the
    //    pivot column's entry becomes -g.  The result is the new panel E + I on P.
    // published record: [pivot row columns p+1 .. p+31 (rotated), 1 / pivot]
    auto publish = [&](double* pn) {
#pragma unroll
      for (int c = 0; c < FNP_NB - 2; c += 2) *reinterpret_cast<double2*>(pn + c) = make_double2(d[c + 1], d[c + 2]);
      if (d[0] == 0.0 || !isfinite(d[0])) s_bad = 1;
      *reinterpret_cast<double2*>(pn + FNP_NB - 2) = make_double2(d[FNP_NB - 1], 1.0 / d[0]);
    };
    double rsc = 1.0;  // scale of this row (1/piv once it has been the pivot)
    if (hasrow && tid == j0) publish(rowbuf);
    for (int p = 0; p < nb; ++p) {
      __syncthreads();
      const double* pr = rowbuf + (p & 1) * FNP_NB;
      double v[FNP_NB];
#pragma unroll
      for (int c = 0; c < FNP_NB; c += 2) {
        const double2 t2 = *reinterpret_cast<const double2*>(pr + c);
        v[c] = t2.x;
        v[c + 1] = t2.y;
      }
      const double inv = v[FNP_NB - 1];
      if (hasrow) {
        // lazy pivot scaling: the pivot row only rotates (gg = 0, its new
        // column is 1) and remembers its scale 1/piv, applied after the panel
        // -- no divergent branch in the step
        const bool ispiv = tid == j0 + p;
        const double gg = ispiv ? 0.0 : d[0] * inv;
        rsc = ispiv ? inv : rsc;
#pragma unroll
        for (int c = 0; c < FNP_NB - 1; ++c) d[c] = fma(-gg, v[c], d[c + 1]);
        d[FNP_NB - 1] = ispiv ? 1.0 : -gg;
        if (p + 1 < nb && tid == j0 + p + 1) publish(rowbuf + ((p + 1) & 1) * FNP_NB);  // next pivot: d[0]
      }
    }
    FNP_MARK(3);
    // c) E -> Es (E = new panel - I on P); d) owner: new panel columns.
    //    After nb steps d[c] holds column (c + nb) mod 32.
    if (hasrow) {
#pragma unroll
      for (int c = 0; c < FNP_NB; ++c) {
        const int col = (c + nb) & (FNP_NB - 1);
        const double x = d[c] * rsc;
        Es[(size_t)col * ldn + tid] = x - (tid == j0 + col ? 1.0 : 0.0);
        if (owner && col < nb) slice[(size_t)(j0 - c0 + col) * ldn + tid] = x;
      }
    }
    const int pt0 = j0 >> 3, pt1 = (j0 + nb + 7) >> 3;
    __syncthreads();
    FNP_MARK(4);
    // e) A[:, own rest] += E * A[P, own rest].  A warp keeps its row tile's E
    //    fragments in registers and sweeps the column tiles four at a time
    //    (independent accumulators).  Rows outside P first (they read the P
    //    rows in place), then the P rows (all reads before any write).  Column
    //    tiles [lo, hi) minus the current panel's and minus [x0, x1).
    const int pc0 = owner ? (j0 - c0) >> 3 : -1, pc1 = owner ? (j0 - c0 + nb + 7) >> 3 : -1;
    const int trow = min(j0 + tq, ldn - 1);  // B operand row (k-step 0); E is zero past nb
    auto row_tile = [&](int rt, bool store_now, double (*keep)[4][2], int lo, int hi, int x0, int x1) {
      const int r0 = rt * 8;
      double a[FNP_NB / 4];
#pragma unroll
      for (int ks = 0; ks < FNP_NB / 4; ++ks) a[ks] = Es[(size_t)(4 * ks + tq) * ldn + r0 + g];
      for (int cb = lo; cb < hi; cb += 4) {
        double acc[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int cc = (cb + u) * 8;
          const bool ok = cb + u < hi;
          acc[u][0] = ok ? slice[(size_t)(cc + 2 * tq) * ldn + r0 + g] : 0.0;
          acc[u][1] = ok ? slice[(size_t)(cc + 2 * tq + 1) * ldn + r0 + g] : 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < FNP_NB / 4; ++ks) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int cc = min(cb + u, hi - 1) * 8;
            const double b = slice[(size_t)(cc + g) * ldn + min(trow + 4 * ks, ldn - 1)];
            dmma_8x8x4(acc[u][0], acc[u][1], a[ks], b);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int ct = cb + u;
          if (ct >= hi || (ct >= pc0 && ct < pc1) || (ct >= x0 && ct < x1)) continue;
          if (store_now) {
            slice[(size_t)(ct * 8 + 2 * tq) * ldn + r0 + g] = acc[u][0];
            slice[(size_t)(ct * 8 + 2 * tq + 1) * ldn + r0 + g] = acc[u][1];
          } else {
            keep[(cb - lo) / 4][u][0] = acc[u][0];
            keep[(cb - lo) / 4][u][1] = acc[u][1];
          }
        }
      }
    };
    auto update_cols = [&](int lo, int hi, int x0, int x1) {
      for (int rt = warp; rt < nrt8; rt += FNP_WARPS)
        if (!(rt >= pt0 && rt < pt1)) row_tile(rt, true, nullptr, lo, hi, x0, x1);
      // P rows: nb/8 <= 4 row tiles, one per warp; <= 16 column tiles -> <= 4 blocks of 4
      double keep[4][4][2];
      const int prt = pt0 + warp;
      const bool pw = prt < pt1;
      __syncthreads();
      if (pw) row_tile(prt, false, keep, lo, hi, x0, x1);
      __syncthreads();
      if (pw) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int ct = lo + q * 4 + u;
            if (ct >= hi || (ct >= pc0 && ct < pc1) || (ct >= x0 && ct < x1)) continue;
            slice[(size_t)(ct * 8 + 2 * tq) * ldn + prt * 8 + g] = keep[q][u][0];
            slice[(size_t)(ct * 8 + 2 * tq + 1) * ldn + prt * 8 + g] = keep[q][u][1];
          }
      }
      __syncthreads();
    };
    update_cols(0, nct, 0, 0);
    FNP_MARK(5);
  }

#ifdef OSPH_FACTOR_PROF
  if (tid == 0 && blockIdx.x == 0)
    printf("factor_np m=%d n=%d CS=%d cycles: gen %lld  export+cluster %lld  import %lld  dinv %lld  E %lld  update %lld\n",
           m, n, CS, _fa[0], _fa[1], _fa[2], _fa[3], _fa[4], _fa[5]);
#endif
  // ---- 3. ||X||_1, tiled X for the sweep, chain constants
  {
    double cmax = 0.0;
    for (int c = warp; c < cw; c += FNP_WARPS) {
      double s = 0.0;
      for (int i = lane; i < n; i += 32) s += fabs(slice[(size_t)c * ldn + i]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      cmax = fmax(cmax, s);
    }
    if (lane == 0 && cw > 0) np_atomic_max_pos(norms + 2 * m + 1, cmax);
  }
  {
    double* Xt = xt_all + xt_off[m];
    const int npad = nrt8 * 8;
    const int cend = (c1 == n) ? (n + OSPH_TILE_KC - 1) / OSPH_TILE_KC * OSPH_TILE_KC : c1;
    // column c of X (pivot order) is column perm[c] of X P^T (natural ring
    // order, the sweep's operand); the late ring's column (perm = 0) is zero
    for (int c = c0 + warp; c < cend; c += FNP_WARPS) {
      const int cn = c < n ? __ldg(perm + c) : c;
      for (int i = lane; i < npad; i += 32)
        Xt[tile_index(i, cn, nrt8)] = (i < n && c < n && cn != 0) ? slice[(size_t)(c - c0) * ldn + i] : 0.0;
    }
    const int jl = pinv[0];  // w_m = X[:, j*], the late ring's column
    if (jl >= c0 && jl < c1)
      for (int i = tid; i < n; i += FNP_THREADS) w_out[(size_t)m * uw_ld(L) + i] = slice[(size_t)(jl - c0) * ldn + i];
  }
  if (tid == 0 && s_bad) atomicOr(status_out + m, 1);
  cluster.sync();  // the below-block rows of every rank are in global memory
  // u_m[j] = Pb_m[ring m-1, :] . X[:, j] for own columns, stored in natural ring
  // order: the sweep's chain partial a_{m-1} = Pb_m[m-1, :] . x'_m is u_m . rhs_m
  {
    double* u = u_out + (size_t)m * uw_ld(L);
    const double* Pb = pbelow + pb_off[m];
    const int nrtpb = (m + 7) >> 3;
    for (int c = warp; c < cw; c += FNP_WARPS) {
      double s = 0.0;
      if (m >= 1)
        for (int l = lane; l < n; l += 32) s += __ldcg(Pb + tile_index(m - 1, l, nrtpb)) * slice[(size_t)c * ldn + l];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        const int cn = __ldg(perm + c0 + c);  // natural ring order; the late ring's weight is zero
        u[cn] = cn != 0 ? s : 0.0;
      }
    }
  }
  const int js = pinv[0];
  if (js >= c0 && js < c1) {  // owner of column j* (ring m): beta_m = Pb_m[m-1, :] . X[:, j*]
    double acc = 0.0;
    if (m >= 1) {
      const double* Pb = pbelow + pb_off[m];
      const int nrtpb = (m + 7) >> 3;
      for (int l = tid; l < n; l += FNP_THREADS)
        acc += __ldcg(Pb + tile_index(m - 1, l, nrtpb)) * slice[(size_t)(js - c0) * ldn + l];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) s_red[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double b = 0.0;
      for (int w = 0; w < FNP_WARPS; ++w) b += s_red[w];
      beta_out[m] = b;
      jstar_out[m] = js;
    }
  }
}

size_t factor_np_smem(int nmax, int cs) { return sizeof(double) * NpLayout(nmax, cs).total_doubles; }

// Launch the static-pivot factorisation for orders m_first..m_last (block
// sizes n <= nmax, nmax <= 256), cs CTAs per order.
cudaError_t launch_factor_np_class(osph_plan* p, int m_first, int m_last, int cs, cudaStream_t st) {
  const int L = p->L;
  const int nmax = L - m_first;
  const size_t smem = factor_np_smem(nmax, cs);
  cudaError_t e = cudaFuncSetAttribute(k_factor_np, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cs > 8 && (e = cudaFuncSetAttribute(k_factor_np, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((m_last - m_first + 1) * cs));
  cfg.blockDim = dim3(FNP_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, k_factor_np, L, m_first, nmax, (const double*)p->d_cos, (const double2*)p->d_rec,
                         (const int*)p->d_ls, (const double2*)p->d_pstart, (const int*)p->d_piv, p->d_xt,
                         (const int64_t*)p->d_xt_off, p->d_pbelow, (const int64_t*)p->d_pb_off, p->d_panel,
                         p->d_norms, p->d_status, p->d_jstar, p->d_beta, p->d_u, p->d_w);
  p->launches++;
  return e;
}
