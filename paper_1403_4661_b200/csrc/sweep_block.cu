// sweep_block.cu -- the order-peeling sweep, peeled a BLOCK of orders at a time
// (the default at L <= 512, for every batch size).
//
// Reference recurrence (pkg/src/optisph/transform.py:441-463): for
// s = L-1 .. 0 solve order s, then subtract its aliases from every ring k < s.
// A correction of order s on ring k lands on the right-hand side of order
//   tm = |+-s mod (2k+1)|   (the same or the opposite tone),
// and for the rings just below s that is the principal alias tm = 2k+1-s:
// ring k = s-1-r corrects entry r of order s-2r-1.  So inside a block of
// OSPH_SB_BLOCK = 32 consecutive orders only the first 16 right-hand-side
// entries of an order depend on orders of the same block, through the 16 rings
// just below each source order.  With U_s = Pb_s[rings s-16..s-1, :] X_s
// (written by the factorisation, factor_bf.cu k_bf_couple) the correction
// order s sends through ring s-1-r is
//   c_s[r] = U_s[r, :] g~_s = U_s[r, :] g_s - sum_j U_s[r, j] d_s[j],
// g_s the right-hand side corrected by every order ABOVE the block and d_s the
// in-block corrections it has received -- a scalar recurrence over the block
// (k_sb_chain) that needs only the small products a_s = U_s g_s.  A block is
//   1. a_s = U_s g_s                 k_sb_gemm<2>, one launch over every order of the block
//                                    (it also merges the pending R2 into R, see below)
//   2. the scalar recurrence; R[s][j] -= d_s[j]                        k_sb_chain
//   3. x_s = X_s g~_s                k_sb_gemm<0>, one launch (-> flm and the block's x buffer)
//   4. G_s = Pb_s x_s, rings k < s   k_sb_gemm<1>, one launch, reduced straight into the
//                                    right-hand sides of the orders below the block
// instead of two launches per order: the L sequential steps of the reference
// loop become L/32 block steps of whole-GPU fp64 tensor-core GEMMs
// (mma.sync m8n8k4 -> DMMA.8x8x4).
//
// Bitwise reproducibility.  Inside one launch of step 4 (32 consecutive orders)
// two corrections can meet in one bin of a ring k >= 16 only as a same-tone /
// opposite-tone pair (s' = -s mod 2k+1, since 2k+1 > 32).  The same-tone branch
// reduces into R, the opposite-tone branch into a second array R2 that the
// next visit of those rows adds in: every address takes at most one reduction
// per launch and launches are ordered.  The short rings k < 16 (where several
// sources can meet) are written out and gathered per target in a fixed order
// by k_sb_combine before the final block, where all of their targets live.
//
// The final block (orders < 32) keeps every ring below each order in U_s, so
// all of its aliases (any tm, including bin 0) are resolved by the recurrence.
// Blocks start at multiples of 32, so a block with m0 >= 32 has no in-block
// alias other than the principal one (the next alias of order m is >= 3m+1).
#include <algorithm>
#include <cstdlib>

#include "plan.cuh"

#define SB_THREADS 256
#define SB_KC 32
#define SB_B OSPH_SB_BLOCK

__device__ __forceinline__ uint32_t sb_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sb_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sb_smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void sb_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void sb_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// alias target of order s on ring k for tone `slot` (transform.py:459-463; bin 0: the - tone
// goes to order 0's - slot, folded into the + slot before order 0 is solved)
__device__ __forceinline__ void sb_target(int s, int k, int slot, int& tm, int& ts) {
  const int nk = 2 * k + 1, rr = s % nk;
  if (rr == 0) {
    tm = 0;
    ts = slot;
  } else if (rr <= k) {
    tm = rr;
    ts = slot;
  } else {
    tm = nk - rr;
    ts = slot ^ 1;
  }
}

template <int TM, int MAPS, bool MERGE = false>
struct SbStage {
  double a[TM / 8][SB_KC][8];  // row tiles as stored: [k][row % 8]
  double b[MAPS][SB_KC][4];    // [map][k][+re, +im, -re, -im]
  double b2[MERGE ? MAPS : 1][MERGE ? SB_KC : 1][4];  // MODE 2: the same rows of R2 (merged into R)
};

// One GEMM per order s = s_top - blockIdx.z of the block, CTA tile TM rows x MAPS maps.
// MODE 0  solve:       A = X_s tiles, rows = degrees, K = rings; B = R slab of order s
// MODE 1  corrections: A = Pb_s tiles, rows = rings k < s, K = degrees; B = the block's x buffer
// MODE 2  coupling:    A = U_s tiles, rows r < min(sb_rows(s), s), K = rings; B = R slab
template <int MODE, int NS, int TM, int MAPS>
__global__ void __launch_bounds__(SB_THREADS) k_sb_gemm(int L, int s_top, int m0, int B,
                                                        const double* __restrict__ atiles,
                                                        const int64_t* __restrict__ a_off,
                                                        const double* __restrict__ w_all, double2* __restrict__ R,
                                                        double2* __restrict__ R2, double2* __restrict__ xblk,
                                                        double2* __restrict__ out, double2* __restrict__ flm) {
  pdl_start();
  extern __shared__ __align__(16) unsigned char sb_raw[];
  using Stage = SbStage<TM, MAPS, MODE == 2>;
  Stage* st = reinterpret_cast<Stage*>(sb_raw);
  const int z = blockIdx.z, s = s_top - z;
  const int n = L - s;
  const int M = MODE == 0 ? n : MODE == 1 ? s : min(sb_rows(s), s);  // output rows
  const int rt0 = blockIdx.x * (TM / 8);                            // first 8-row tile
  if (rt0 * 8 >= M && !(MODE == 2 && rt0 == 0)) return;  // MODE 2 also merges R2 into R: every order's rows
  const int nrt = MODE == 0 ? (n + 7) >> 3 : MODE == 1 ? (s + 7) >> 3 : sb_rows(s) >> 3;
  const int b0 = blockIdx.y * MAPS;
  const double* A = atiles + __ldg(a_off + s);
  const int64_t npos = (int64_t)L * (L + 1) / 2, p0 = packed_pos(L, s, 0);
  const double2* xz = xblk + (int64_t)z * B * 2 * L;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int nch = (n + SB_KC - 1) / SB_KC;

  auto load = [&](int buf, int c) {
    Stage& S = st[buf];
    for (int i = tid; i < (TM / 8) * 128; i += SB_THREADS) {  // 128 16-byte pieces per 8-row tile
      const int t = i >> 7, q = i & 127;
      double* dst = &S.a[t][0][0] + 2 * q;
      if (rt0 + t < nrt) sb_cp16(dst, A + ((int64_t)c * nrt + rt0 + t) * 256 + 2 * q);
      else *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
    }
    for (int i = tid; i < MAPS * SB_KC * 2; i += SB_THREADS) {
      const int mp = i / (SB_KC * 2), rem = i % (SB_KC * 2), k = rem >> 1, slot = rem & 1;
      const int kk = c * SB_KC + k, b = b0 + mp;
      double* dst = &S.b[mp][k][2 * slot];
      if (kk < n && b < B) {
        const int64_t ri = ((int64_t)b * npos + p0 + kk) * 2 + slot;
        const double2* src = MODE == 1 ? xz + ((int64_t)b * 2 + slot) * L + kk : R + ri;
        sb_cp16(dst, src);
        if (MODE == 2) sb_cp16(&S.b2[mp][k][2 * slot], R2 + ri);
      } else {
        *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
        if (MODE == 2) *reinterpret_cast<double2*>(&S.b2[mp][k][2 * slot]) = make_double2(0.0, 0.0);
      }
    }
    sb_commit();
  };

  // warps: WCG column groups of 16 (2 blocks of 8) x WRG row groups of RB blocks of 8
  constexpr int WCG = MAPS / 4, WRG = 8 / WCG, RB = TM / (8 * WRG);
  static_assert(WCG * WRG == 8 && RB >= 1 && RB * 8 * WRG == TM, "CTA tile does not map onto 8 warps");
  const int wr = (warp % WRG) * (TM / WRG), wc = (warp / WRG) * 16;
  double acc[RB][2][2];
#pragma unroll
  for (int i = 0; i < RB; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int c = 0; c < NS - 1; ++c) {
    if (c < nch) load(c, c);
    else sb_commit();
  }
  for (int c = 0; c < nch; ++c) {
    sb_wait<NS - 2>();
    __syncthreads();  // chunk c visible to all; stage (c - 1) % NS free
    if (c + NS - 1 < nch) load((c + NS - 1) % NS, c + NS - 1);
    else sb_commit();
    Stage& S = st[c % NS];
    if (MODE == 2) {
      // The opposite-tone corrections of the blocks above wait in R2 (k_sb_gemm<1>): this
      // launch visits every right-hand-side row of the block exactly once (grid.x = 1), so it
      // adds them in -- R += R2, R2 = 0 in global memory for the solve that follows, and in
      // the staged operand for its own products.
      for (int i = tid; i < MAPS * SB_KC * 2; i += SB_THREADS) {
        const int mp = i / (SB_KC * 2), rem = i % (SB_KC * 2), k = rem >> 1, slot = rem & 1;
        const double2 v2 = *reinterpret_cast<const double2*>(&S.b2[mp][k][2 * slot]);
        if (v2.x != 0.0 || v2.y != 0.0) {
          double2* bp = reinterpret_cast<double2*>(&S.b[mp][k][2 * slot]);
          const double2 v = make_double2(bp->x + v2.x, bp->y + v2.y);
          *bp = v;
          const int64_t ri = ((int64_t)(b0 + mp) * npos + p0 + c * SB_KC + k) * 2 + slot;
          R[ri] = v;
          R2[ri] = make_double2(0.0, 0.0);
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int k0 = 0; k0 < SB_KC; k0 += 4) {
      double a[RB], b[2];
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int row = wr + 8 * i + g;
        a[i] = S.a[row >> 3][k0 + tq][row & 7];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = wc + 8 * j + g;  // map col >> 2, component col & 3
        b[j] = S.b[col >> 2][k0 + tq][col & 3];
      }
#pragma unroll
      for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }

  const double sg = (s & 1) ? -1.0 : 1.0;
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    const int row = rt0 * 8 + wr + 8 * i + g;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (row >= M) continue;
      const int col = wc + 8 * j + 2 * tq;  // even: (re, im) of one (map, slot)
      const int mp = col >> 2, slot = (col >> 1) & 1, b = b0 + mp;
      if (b >= B) continue;
      double vr = acc[i][j][0], vi = acc[i][j][1];
      if (MODE == 0) {
        // late ring's column (zeroed in the X tiles): + w[row] * rhs[0]
        const double w = __ldg(w_all + (int64_t)s * uw_ld(L) + row);
        const double2 g0 = R[((int64_t)b * npos + p0) * 2 + slot];
        vr = fma(w, g0.x, vr);
        vi = fma(w, g0.y, vi);
        if (slot) {
          vr *= sg;
          vi *= sg;
        }
        const double2 x = make_double2(vr, vi);
        xblk[(int64_t)z * B * 2 * L + ((int64_t)b * 2 + slot) * L + row] = x;
        const int64_t ell = s + row;
        double2* f = flm + (int64_t)b * L * L + ell * ell + ell;
        if (slot == 0) f[s] = x;
        else if (s > 0) f[-s] = x;
      } else if (MODE == 1) {
        if (slot) {  // G_-s carries (-1)^s
          vr *= sg;
          vi *= sg;
        }
        // Alias target of ring k = row.  Inside one launch (32 consecutive orders) two
        // corrections meet in one bin only as a same-tone / opposite-tone pair
        // (s' = -s mod 2k+1) once 2k+1 > 32, so the same-tone branch reduces into R and the
        // opposite-tone branch into R2 (added to R before the target's block starts,
        // k_sb_combine): every address takes at most one reduction per launch and the
        // sums are bitwise reproducible.  Rings k < 16 go through `out` (gathered by k_sb_combine
        // before the final block, where all of their targets live).
        const int k = row;
        if (k < SB_B / 2) {
          out[(((int64_t)z * (SB_B / 2) + k) * B + b) * 2 + slot] = make_double2(vr, vi);
        } else {
          const int nk = 2 * k + 1, rr = s % nk;
          const bool same = rr <= k;  // rr == 0: bin 0, the tone keeps its slot
          const int tm = same ? rr : nk - rr, ts = same ? slot : slot ^ 1;
          if (tm < m0) {  // targets inside the block were resolved by k_sb_chain
            double2* rp = (same ? R : R2) + ((int64_t)b * npos + packed_pos(L, tm, k - tm)) * 2 + ts;
            atomicAdd(&rp->x, -vr);
            atomicAdd(&rp->y, -vi);
          }
        }
      } else {
        out[(((int64_t)z * SB_B + row) * B + b) * 2 + slot] = make_double2(vr, vi);
      }
    }
  }
}

// The in-block recurrence.  Block = orders m0 .. s_top (nb <= 32).  JR = rows of U per
// order (16; 32 in the final block) = right-hand-side entries that can take an in-block
// correction.  A map is handled by 4 JR threads = (row, tone, re/im), whole warps that
// synchronise among themselves only (named barrier per map); a CTA holds 256 / (4 JR) maps.
// Shared memory per map: delta[z][j][tone][re/im], the in-block corrections of entry j of
// order s_top - z, and a[z][r][tone][re/im], the coupling products (loaded once).  The
// coefficients U_s[r, 0..JR) of the next order are prefetched into registers.  Per source
// order s (descending), row r (ring k = s-1-r): c = a_s[r] - sum_j U_s[r, j] delta_s[j] is
// added to the target's delta.  Sources are processed in order and the targets of one
// source are distinct, so every sum has a fixed order.  Finally R[s][j] -= delta_s[j].
template <int JR>
__global__ void __launch_bounds__(SB_THREADS) k_sb_chain(int L, int s_top, int m0, int B,
                                                         const double* __restrict__ ut,
                                                         const int64_t* __restrict__ ut_off,
                                                         const double2* __restrict__ abuf, double2* __restrict__ R) {
  pdl_start();
  constexpr int TPM = 4 * JR, MAPS = SB_THREADS / TPM;  // threads per map, maps per CTA
  constexpr bool USM = JR == SB_B / 2;                   // U blocks of the whole block in shared memory (64 KB)
  extern __shared__ __align__(16) double sm_chain[];
  __shared__ int64_t uoff[SB_B];
  const int nb = s_top - m0 + 1;
  const int tid = threadIdx.x, mp = tid / TPM, t = tid - mp * TPM;
  const int comp = t & 1, slot = (t >> 1) & 1, c4 = t & 3, rl = t >> 2;  // rl < JR
  double* delta = sm_chain + (size_t)mp * (2 * SB_B * JR * 4);  // [nb][JR][4]
  double* asm_ = delta + SB_B * JR * 4;                         // [nb][JR][4]
  double* usm = sm_chain + (size_t)MAPS * (2 * SB_B * JR * 4);  // USM: [nb][JR / 8][JR][8]
  const int b = blockIdx.x * MAPS + mp;
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  if (tid < nb) uoff[tid] = __ldg(ut_off + (s_top - tid));
  // a[z][r][tone][re/im] of this map: 32 contiguous bytes per (z, r), copied asynchronously
  for (int i = t; i < nb * JR * 2; i += TPM) {
    const int sl = i & 1, zr = i >> 1, r = zr % JR, z = zr / JR;
    double* dst = asm_ + (size_t)zr * 4 + 2 * sl;
    if (b < B && r < min(sb_rows(s_top - z), s_top - z)) sb_cp16(dst, abuf + (((int64_t)z * SB_B + r) * B + b) * 2 + sl);
    else *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
  }
  for (int i = t; i < nb * JR * 4; i += TPM) delta[i] = 0.0;
  __syncthreads();
  if (USM) {  // first JR columns of every order's JR / 8 row tiles: JR * 8 contiguous doubles each
    for (int i = tid; i < nb * (JR / 8) * JR * 4; i += SB_THREADS) {
      const int q = i % (JR * 4), zt = i / (JR * 4), tt = zt % (JR / 8), z = zt / (JR / 8);
      if (s_top - z >= 1) sb_cp16(usm + (size_t)zt * JR * 8 + 2 * q, ut + uoff[z] + tt * 256 + 2 * q);
    }
  }
  sb_commit();
  sb_wait<0>();
  __syncthreads();
  auto group_sync = [&]() { asm volatile("bar.sync %0, %1;\n" ::"r"(1 + mp), "r"(TPM) : "memory"); };
  double un[USM ? 1 : JR];  // !USM: U_s[rl, 0..JR) of the order about to be processed (register prefetch)
  auto u_fetch = [&](int z) {
    if (USM) return;
    const int s = s_top - z;
    const bool ok = z < nb && s >= 1 && rl < min(sb_rows(s), s);
    const double* ur = ut + (z < nb ? uoff[z] : 0) + (rl >> 3) * 256 + (rl & 7);
#pragma unroll
    for (int j = 0; j < (USM ? 1 : JR); ++j) un[j] = ok ? __ldg(ur + j * 8) : 0.0;
  };
  u_fetch(0);
  for (int z = 0; z < nb; ++z) {
    double u[JR];
    if (USM) {
      const double* ur = usm + ((size_t)z * (JR / 8) + (rl >> 3)) * JR * 8 + (rl & 7);
#pragma unroll
      for (int j = 0; j < JR; ++j) u[j] = ur[j * 8];
    } else {
#pragma unroll
      for (int j = 0; j < JR; ++j) u[j] = un[USM ? 0 : j];
      u_fetch(z + 1);
    }
    const int s = s_top - z;
    const int rows = min(sb_rows(s), s);
    if (rl < rows) {
      const int r = rl, k = s - 1 - r;
      int tm, ts;
      if (JR == SB_B / 2) {  // m0 >= 32 > r: 2k+1 > s, the principal alias
        tm = s - 2 * r - 1;
        ts = slot ^ 1;
      } else {
        sb_target(s, k, slot, tm, ts);
      }
      if (tm >= m0 && k - tm < JR) {
        const double* dz = delta + (size_t)z * JR * 4 + c4;
        double c0 = asm_[((size_t)z * JR + r) * 4 + c4], c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll
        for (int j = 0; j < JR; j += 4) {  // entries past n_s and untouched entries hold zero
          c0 = fma(-u[j], dz[j * 4], c0);
          c1 = fma(-u[j + 1], dz[(j + 1) * 4], c1);
          c2 = fma(-u[j + 2], dz[(j + 2) * 4], c2);
          c3 = fma(-u[j + 3], dz[(j + 3) * 4], c3);
        }
        delta[((size_t)(s_top - tm) * JR + (k - tm)) * 4 + ((ts << 1) | comp)] += (c0 + c1) + (c2 + c3);
      }
    }
    group_sync();  // delta of the next order complete
  }
  // apply R[s][j] -= delta_s[j]: independent read-modify-writes, sixteen in flight per thread.
  // Thread rl owns entry j = rl of every order; in a block above the final one order z can
  // only have received corrections in entries j <= (z - 1) / 2.
  if (b < B) {
    const int z_lo = JR == SB_B / 2 ? 2 * rl + 1 : 0;
    for (int z0 = z_lo; z0 < nb; z0 += 16) {
      int64_t ri[16];
      double d[16], v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int z = z0 + q, m = s_top - z;
        ri[q] = -1;
        d[q] = 0.0;
        if (z < nb && rl < L - m) {
          d[q] = delta[((size_t)z * JR + rl) * 4 + c4];
          if (d[q] != 0.0) ri[q] = (((int64_t)b * npos + packed_pos(L, m, rl)) * 2 + slot) * 2 + comp;
        }
      }
      double* Rd = reinterpret_cast<double*>(R);
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = ri[q] >= 0 ? __ldcg(Rd + ri[q]) : 0.0;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (ri[q] >= 0) Rd[ri[q]] = v[q] - d[q];
    }
  }
}

// R += R2 over the rows of a ONE-order block (orders m0 = s_top; otherwise the coupling
// launch k_sb_gemm<2> merges them): grid (x, B), map blockIdx.y.
__global__ void __launch_bounds__(256) k_sb_merge(int L, int s_top, int m0, double2* __restrict__ R,
                                                  double2* __restrict__ R2) {
  pdl_start();
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  const int64_t p_lo = packed_pos(L, m0, 0) * 2, per = packed_pos(L, s_top + 1, 0) * 2 - p_lo;
  double2* rp = R + (int64_t)blockIdx.y * npos * 2 + p_lo;
  double2* r2 = R2 + (int64_t)blockIdx.y * npos * 2 + p_lo;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = r2[i];
    if (v.x != 0.0 || v.y != 0.0) {
      const double2 r = rp[i];
      rp[i] = make_double2(r.x + v.x, r.y + v.y);
      r2[i] = make_double2(0.0, 0.0);
    }
  }
}

// Before the final block (orders < 32): the corrections every block above sent through the
// short rings k < 16 (several sources can meet in one bin there; their targets, orders
// tm <= k < 16, all belong to the final block).  k_sb_gemm<1> left them in G16, one slice of
// [32 sources][16 rings][B][tone] per block.  One warp per target (ring k, order tm <= k,
// tone ts, map b): 136 (k, tm) pairs x 2 tones; blocks from the top down, lane = source
// order s_top - lane of the block; the matching corrections are summed in lane order
// (descending source order; a source sends at most one of its tones to a target).
__global__ void __launch_bounds__(256) k_sb_combine(int L, int B, const double2* __restrict__ G16,
                                                    double2* __restrict__ R) {
  pdl_start();
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  constexpr int NT = (SB_B / 2) * (SB_B / 2 + 1) / 2 * 2;
  const int lane = threadIdx.x & 31;
  const int64_t slice = (int64_t)SB_B * (SB_B / 2) * B * 2;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < (int64_t)NT * B;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int b = (int)(w % B);
    int tt = (int)(w / B);
    const int ts = tt & 1;
    tt >>= 1;
    int k = 0;
    while (tt >= k + 1) {  // tt = k (k + 1) / 2 + tm
      tt -= k + 1;
      ++k;
    }
    const int tm = tt, nk = 2 * k + 1;
    double ax = 0.0, ay = 0.0;
    bool any = false;
    int blk = 0;
    for (int s_top = L - 1; s_top >= SB_B; ++blk) {
      const int m0 = (s_top / SB_B) * SB_B;
      const int s = s_top - lane;
      double2 g = make_double2(0.0, 0.0);
      bool hit = false;
      if (s >= m0 && s > k) {
        const int rr = s % nk;
        const bool same = rr <= k;
        if ((same ? rr : nk - rr) == tm) {
          const int slot = same ? ts : ts ^ 1;  // the tone of source s that lands on tone ts
          g = __ldcg(G16 + blk * slice + (((int64_t)lane * (SB_B / 2) + k) * B + b) * 2 + slot);
          hit = true;
        }
      }
      unsigned mask = __ballot_sync(0xffffffffu, hit);
      any |= mask != 0;
      while (mask) {  // ascending lanes = descending source orders
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        ax += __shfl_sync(0xffffffffu, g.x, src);
        ay += __shfl_sync(0xffffffffu, g.y, src);
      }
      s_top = m0 - 1;
    }
    if (lane == 0 && any) {
      double2* rp = R + ((int64_t)b * npos + packed_pos(L, tm, k - tm)) * 2 + ts;
      const double2 r = *rp;
      *rp = make_double2(r.x - ax, r.y - ay);
    }
  }
}

// R[b][pos(0, k)][+] += R[b][pos(0, k)][-] for every ring k (plain layout).
__global__ void k_sb_fold_order0(int L, double2* __restrict__ R) {
  pdl_start();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  double2* rp = R + ((int64_t)blockIdx.y * npos + k) * 2;  // pos(0, k) = k
  rp[0] = make_double2(rp[0].x + rp[1].x, rp[0].y + rp[1].y);
}

int ensure_sweep_blocked(osph_plan* p) {
  if (p->d_sb_x) return OSPH_OK;
  const size_t L = p->L, B = p->max_batch;
  const size_t nr2 = L * (L + 1) * B;  // [B][pos][+-], like R (plain layout)
  cudaError_t e;
  if ((e = cudaMalloc(&p->d_sb_x, sizeof(double2) * SB_B * B * 2 * L)) != cudaSuccess ||
      (e = cudaMalloc(&p->d_sb_a, sizeof(double2) * SB_B * SB_B * B * 2)) != cudaSuccess ||
      (e = cudaMalloc(&p->d_sb_g, sizeof(double2) * ((L + SB_B - 1) / SB_B) * SB_B * (SB_B / 2) * B * 2)) != cudaSuccess ||
      (e = cudaMalloc(&p->d_sb_r2, sizeof(double2) * nr2)) != cudaSuccess ||
      (e = cudaMemsetAsync(p->d_sb_r2, 0, sizeof(double2) * nr2, p->stream)) != cudaSuccess) {
    osph_set_error(std::string("blocked sweep buffers: ") + cudaGetErrorString(e));
    return OSPH_ERR_CUDA;
  }
  return OSPH_OK;
}

template <int NS, int TM, int MAPS>
static cudaError_t sweep_blocked_run(osph_plan* p, int B, double2* flm, int b0) {
  const int L = p->L;
  // maps b0 .. b0 + B - 1 of the spectra (plain layout [map][pos][+-]); flm is already the first map's
  double2* const Rb = p->d_r + (int64_t)b0 * L * (L + 1);
  double2* const R2b = p->d_sb_r2 + (int64_t)b0 * L * (L + 1);
  const size_t smem = NS * sizeof(SbStage<TM, MAPS>);
  cudaError_t e;
  auto k_solve = k_sb_gemm<0, NS, TM, MAPS>;
  auto k_corr = k_sb_gemm<1, NS, TM, MAPS>;
  auto k_cpl = k_sb_gemm<2, 4, 32, 8>;  // at most 32 coupling rows per order: 32 x 8 maps per CTA
  const size_t smem_cpl = 4 * sizeof(SbStage<32, 8, true>);
  if ((e = cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(k_corr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(k_cpl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cpl)) != cudaSuccess)
    return e;
  // chain kernel shared memory: delta + a of every map of the CTA
  auto chain_smem = [](int JR) {
    return sizeof(double) * ((size_t)(SB_THREADS / (4 * JR)) * 2 * SB_B * JR * 4 +
                             (JR == SB_B / 2 ? (size_t)SB_B * JR * JR : 0));
  };
  if ((e = cudaFuncSetAttribute(k_sb_chain<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chain_smem(16))) !=
          cudaSuccess ||
      (e = cudaFuncSetAttribute(k_sb_chain<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chain_smem(32))) !=
          cudaSuccess)
    return e;
  const int ny = (B + MAPS - 1) / MAPS;
  cudaStream_t st = p->stream;
  int s_top = L - 1, ps_top = -1, next_rng = 0, blk = 0;
  while (s_top >= 0) {
    const int m0 = (s_top / SB_B) * SB_B;  // blocks start at multiples of 32
    const int nb = s_top - m0 + 1;
    const bool last = m0 == 0;
    // split factorisation: the factors of every range this block touches (ranges descend)
    while (p->sweep_waits_ranges && next_rng < p->n_frng && p->bf_rng[next_rng].m_last >= m0) {
      cudaEvent_t ev = next_rng == p->n_frng - 1 ? p->ev[7] : p->ev_f[next_rng];
      if ((e = cudaStreamWaitEvent(st, ev, 0)) != cudaSuccess) return e;
      ++next_rng;
    }
    if (ps_top >= 0 && nb == 1) {  // a one-order block has no coupling launch to merge R2 into R
      const int64_t per = (packed_pos(L, s_top + 1, 0) - packed_pos(L, m0, 0)) * 2;
      const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((per + 255) / 256, 32));
      if ((e = launch_pdl(k_sb_merge, dim3(gx, B), dim3(256), 0, st, L, s_top, m0, Rb, R2b)) != cudaSuccess)
        return e;
      p->launches++;
    }
    if (last && ps_top >= 0) {  // the short-ring corrections of every block above
      if ((e = launch_pdl(k_sb_combine, dim3((272 * B + 7) / 8), dim3(256), 0, st, L, B, (const double2*)p->d_sb_g,
                          Rb)) != cudaSuccess)
        return e;
      p->launches++;
    }
    if (nb > 1) {
      if ((e = launch_pdl(k_cpl, dim3(1, (B + 7) / 8, nb), dim3(SB_THREADS), smem_cpl, st, L, s_top, m0, B,
                          (const double*)p->d_ut, (const int64_t*)p->d_ut_off, (const double*)p->d_w, Rb,
                          R2b, p->d_sb_x, p->d_sb_a, flm)) != cudaSuccess)
        return e;
      if (last)
        e = launch_pdl(k_sb_chain<32>, dim3((B + 1) / 2), dim3(SB_THREADS), chain_smem(32), st, L, s_top, m0, B,
                       (const double*)p->d_ut, (const int64_t*)p->d_ut_off, (const double2*)p->d_sb_a, Rb);
      else
        e = launch_pdl(k_sb_chain<16>, dim3((B + 3) / 4), dim3(SB_THREADS), chain_smem(16), st, L, s_top, m0, B,
                       (const double*)p->d_ut, (const int64_t*)p->d_ut_off, (const double2*)p->d_sb_a, Rb);
      if (e != cudaSuccess) return e;
      p->launches += 2;
    }
    if (last) {  // order 0: fold the - slot (bin-0 -tone corrections) into the + slot
      if ((e = launch_pdl(k_sb_fold_order0, dim3((L + 127) / 128, B), dim3(128), 0, st, L, Rb)) != cudaSuccess)
        return e;
      p->launches++;
    }
    if ((e = launch_pdl(k_solve, dim3((L - m0 + TM - 1) / TM, ny, nb), dim3(SB_THREADS), smem, st, L, s_top, m0, B,
                        (const double*)p->d_xt, (const int64_t*)p->d_xt_off, (const double*)p->d_w, Rb,
                        R2b, p->d_sb_x, p->d_sb_g, flm)) != cudaSuccess)
      return e;
    p->launches++;
    if (!last) {  // the final block's corrections all land inside the block
      if ((e = launch_pdl(k_corr, dim3((s_top + TM - 1) / TM, ny, nb), dim3(SB_THREADS), smem, st, L, s_top, m0, B,
                          (const double*)p->d_pbelow, (const int64_t*)p->d_pb_off, (const double*)p->d_w, Rb,
                          R2b, p->d_sb_x, p->d_sb_g + (int64_t)blk * SB_B * (SB_B / 2) * B * 2, flm)) !=
          cudaSuccess)
        return e;
      p->launches++;
    }
    ++blk;
    ps_top = s_top;
    s_top = m0 - 1;
  }
  p->sweep_waits_ranges = false;
  return cudaGetLastError();
}

// CTA tile: 64 rows x 8 maps; 64 x 4 maps for small batches (10-20% faster up to B = 8;
// OSPH_SB_SMALL=b moves the threshold).  Measured and removed: 128 x 8, 128 x 16 and 64 x 16
// maps (config 2 sweep 0.85 / 0.79 / 0.79 vs 0.71 ms at the time; DESIGN 12).
cudaError_t launch_sweep_blocked(osph_plan* p, int B, double2* flm, int b0) {
  static const int small_b = getenv("OSPH_SB_SMALL") ? atoi(getenv("OSPH_SB_SMALL")) : 8;
  if (B <= small_b) return sweep_blocked_run<4, 64, 4>(p, B, flm, b0);
  return sweep_blocked_run<4, 64, 8>(p, B, flm, b0);
}
