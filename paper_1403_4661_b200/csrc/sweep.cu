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
// Pipelining.  The solution of order s splits as
//   x_s = x'_s + w_s L_s,  x'_s = X_s P rhs_s (late entry zeroed),  w_s = X_s[:, j*_s],
// where L_s, the right-hand-side entry of ring s, is the only entry that
// depends on order s+1.  It follows from a scalar chain
//   G+-_{s+1}(theta_s) = a+-_s + beta_{s+1} L+-_{s+1},  a_s = Pb_{s+1}[s, :] . x'_{s+1},
// so all bulk work of a step is independent of the chain and a step needs ONE
// cluster barrier.  Step t (t = L-1 .. 0):
//   (a) chain -> L_t                                 (shared memory only)
//   (b) x_t = x'_t + w_t L_t on own rows -> flm and the team exchange buffer (global)
//   (c) CORR(t+1): corrections of order t+1 (x_{t+1} complete) on own rings
//   (d) BULK(t-1): x'_{t-1} on own rows, chain partial a_{t-2} -> DSMEM
// x'_s is computed one step before it is used; the corrections of order s+1
// are applied one step after x_{s+1} is known -- both fit the alias
// dependency structure (orders >= s+3 feed the non-late entries of order s).
//
// Streaming.  CORR and BULK are row-sliced GEMMs (rows of the team split
// over its CTAs, K = n) on the fp64 tensor cores (mma.sync m8n8k4 ->
// DMMA.8x8x4).  Their A operands (8-row tiles of Pb_s / X_s, written by
// factor.cu) do not depend on the data, so one producer thread streams them
// with bulk async copies (cp.async.bulk + mbarrier complete_tx, the TMA
// engine) through an S-stage ring that runs ahead across jobs and steps;
// only the small B operands (x, gathered right-hand sides) wait on the chain.
//
// A "team" = one thread-block cluster owning a group of maps; teams are
// independent, so a batch fills the GPU with teams and a single map gets one
// wide team.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "plan.cuh"

namespace cg = cooperative_groups;

#define SWEEP_THREADS 256
#define SWEEP_WARPS 8
#define SWEEP_IPW 4     // max accumulator tiles per warp
#define SWEEP_UMAX 8    // max gathered right-hand-side entries per thread
#define SWEEP_KC 32     // K columns per streamed chunk
#define SWEEP_SMAX 6    // ring stages: deeper rings measured slower (L=256: S=9 +13%)
#ifndef SWEEP_MINB
#define SWEEP_MINB 1    // resident CTAs per SM the register budget is sized for
#endif

// ---------------------------------------------------------------------------
// mbarrier / bulk-copy PTX

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
// barrier among the 8 consumer warps only (the producer warp never joins it)
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }

// -DOSPH_SWEEP_PROF: per-phase cycle counts of CTA 0 (debug builds only)
#ifdef OSPH_SWEEP_PROF
#define PROF_N 9
#define PROF_DECL            \
  long long _pt = clock64(); \
  long long _acc[PROF_N] = {};
#define PROF_MARK(i)                \
  do {                              \
    consumers_sync();               \
    const long long _n = clock64(); \
    _acc[i] += _n - _pt;            \
    _pt = _n;                       \
  } while (0)
#define PROF_DUMP()                                                                                           \
  if (blockIdx.x == 0 && threadIdx.x == 0)                                                                    \
  printf("sweep prof (cycles): issue %lld chain %lld axpy %lld corr-wait %lld corr %lld bulk-wait %lld "      \
         "bulk-gemm %lld bulk-rest %lld barrier %lld\n",                                                      \
         _acc[0], _acc[1], _acc[2], _acc[3], _acc[4], _acc[5], _acc[6], _acc[7], _acc[8])
#else
#define PROF_DECL
#define PROF_MARK(i)
#define PROF_DUMP()
#endif

#define SWEEP_THREADS_ALL (SWEEP_THREADS + 32)  // + one producer warp


// ---------------------------------------------------------------------------
// configuration and shared-memory layout

struct SweepCfg {
  int L, T, CC, KC, S;
  int tpc;  // max 8-row tiles of one job on one CTA
  int ldx, ldr, ccp;
  size_t xrow, gst, xp, wv, prow, apart, late, rch, stage, bar, total;  // offsets in doubles
  __host__ __device__ SweepCfg(int L_, int T_, int CC_, int KC_, int S_) : L(L_), T(T_), CC(CC_), KC(KC_), S(S_) {
    tpc = ((L + 7) / 8 + T - 1) / T;
    ldx = ((L + 31) / 32) * 32;  // rows of the B operands: every chunk of 32 K-rows is in bounds
    ldr = 8 * tpc + 4;
    // row pitch of the row-major B operands: > CC (column CC stays zero) and
    // = 4 mod 8 doubles, so the (tq, g) lanes of a DMMA B fragment hit distinct banks
    ccp = ((CC + 1 + 3) / 8) * 8 + 4;
    size_t o = 0;
    xrow = o;  o += (size_t)ldx * ccp;          // x_{t+1} of the whole team, row-major [l][ccp] (CORR B)
    gst = o;   o += (size_t)ldx * ccp;          // gathered right-hand side, row-major [j][ccp] (BULK B)
    xp = o;    o += (size_t)2 * CC * ldr;       // own rows of x'_s, transposed, by parity of s
    wv = o;    o += (size_t)2 * ldr;            // own rows of w_s, by parity of s
    prow = o;  o += (size_t)2 * ldr;            // own entries of Pb_s[s-1, :], by parity of s
    apart = o; o += (size_t)4 * T * CC;         // chain partials a_s from every rank, slot s % 4
    late = o;  o += (size_t)2 * CC;             // late right-hand-side entries L_s, by parity
    rch = o;   o += (size_t)2 * CC;             // prefetched R(+-)[s][0], by parity
    o = (o + 15) & ~(size_t)15;                 // 128-byte aligned stages
    stage = o; o += (size_t)S * tpc * KC * 8;
    bar = o;   o += (size_t)2 * S;              // full[S], empty[S]
    total = o;
  }
};

// Job = one row-sliced GEMM of a step.  type 0: BULK(s) (A = X_s tiles),
// type 1: CORR(s) (A = Pb_s tiles, rings k < s-1).
struct Job {
  int type, s, K;   // K = n_s
  int rt0, rt1;     // own 8-row tiles
  int nch;          // chunks of KC columns (0 = nothing to do on this CTA)
  const double* A;  // operand base (X tiles or Pb tiles)
  int64_t off;      // this CTA's row-tile range inside chunk 0 (chunk-major tiles, common.cuh)
  int64_t cstride;  // doubles between consecutive chunks
};

__device__ __forceinline__ Job make_job(int type, int s, int L, int T, int rank, int KC, const double* xt,
                                        const int64_t* xt_off, const double* pbt, const int64_t* pb_off,
                                        bool with_offset) {
  Job j;
  j.type = type;
  j.s = s;
  j.K = L - s;
  const int rows = type == 0 ? j.K : s - 1;  // CORR skips ring s-1 (the chain)
  const int mrows = type == 0 ? j.K : s;     // rows of the stored matrix
  const int nt = (rows + 7) / 8;
  j.rt0 = (rank * nt) / T;
  j.rt1 = ((rank + 1) * nt) / T;
  j.nch = (j.rt1 > j.rt0 && rows > 0) ? (j.K + KC - 1) / KC : 0;
  j.cstride = (int64_t)((mrows + 7) / 8) * KC * 8;
  j.A = type == 0 ? xt : pbt;
  j.off = with_offset ? (type == 0 ? xt_off[s] : pb_off[s]) + (int64_t)j.rt0 * KC * 8 : 0;
  return j;
}

// Job sequence: BULK(L-1) (prologue), then per step t = L-1..0:
// CORR(t+1) if 1 <= t <= L-2, BULK(t-1) if t >= 1.  Cursor (t, ph).
__device__ __forceinline__ bool next_job_id(int L, int& t, int& ph, int& type, int& s) {
  while (t >= 0) {
    if (ph == 0) {
      ph = 1;
      if (t >= 1 && t <= L - 2) {
        type = 1;
        s = t + 1;
        return true;
      }
    } else {
      const int tt = t;
      ph = 0;
      --t;
      if (tt >= 1) {
        type = 0;
        s = tt - 1;
        return true;
      }
    }
  }
  return false;
}

// One job's chunk loop for a warp owning NM output tiles (8x8 each), with
// NCH independent accumulator chains per tile for DMMA latency hiding.
template <int NM, int CC>
__device__ __forceinline__ void job_tiles(int nch, int ldb, const double* stages, size_t stage_elems, uint64_t* full,
                                          uint64_t* empty, int S, int& cst, uint32_t& cphase, const int* aoff,
                                          const int* boff, const double* Bsrc, int tq, int lane,
                                          double (&out)[SWEEP_IPW][2]) {
  constexpr int CH = NM == 1 ? 4 : 2;
  double acc[NM][CH][2];
#pragma unroll
  for (int u = 0; u < NM; ++u)
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[u][c][0] = acc[u][c][1] = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    mbar_wait(full + cst, cphase);
    const double* sA = stages + cst * stage_elems + tq * 8;
    const double* Bk = Bsrc + (size_t)(ch * SWEEP_KC + tq) * ldb;  // row-major B: [k][column]
    // columns past K are zero in the tiled operand and finite in Bsrc: no guard
#pragma unroll
    for (int ks = 0; ks < SWEEP_KC / 4; ++ks) {
#pragma unroll
      for (int u = 0; u < NM; ++u) {
        const double a = sA[aoff[u] + ks * 32];
        const double b = Bk[(size_t)ks * 4 * ldb + boff[u]];
        dmma_8x8x4(acc[u][ks % CH][0], acc[u][ks % CH][1], a, b);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + cst);
    if (++cst == S) {
      cst = 0;
      cphase ^= 1u;
    }
  }
#pragma unroll
  for (int u = 0; u < NM; ++u) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      s0 += acc[u][c][0];
      s1 += acc[u][c][1];
    }
    out[u][0] = s0;
    out[u][1] = s1;
  }
}

template <int CC>
__global__ void __launch_bounds__(SWEEP_THREADS_ALL, SWEEP_MINB) k_sweep(
    int L, int B, int maps_per_team, int KC, int S, const double* __restrict__ xt, const int64_t* __restrict__ xt_off,
    const int* __restrict__ perm_all, const int* __restrict__ jstar_all, const double* __restrict__ beta_all,
    const double* __restrict__ pbt, const int64_t* __restrict__ pb_off, double2* __restrict__ R,
    double2* __restrict__ flm, double* __restrict__ xg_all) {
  cg::cluster_group cluster = cg::this_cluster();
  const int T = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int team = (int)(blockIdx.x / T);
  const int b0 = team * maps_per_team;
  const int gm = min(maps_per_team, B - b0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  constexpr int NCT = (CC + 7) / 8;
  constexpr int NB4 = CC / 4;  // map slots of the team
  const bool producer = warp == SWEEP_WARPS;

  extern __shared__ __align__(128) double smem[];
  const SweepCfg cfg(L, T, CC, KC, S);
  const int ldr = cfg.ldr, tpc = cfg.tpc, ccp = cfg.ccp;
  double* xrow = smem + cfg.xrow;
  double* gst = smem + cfg.gst;
  double* xg = xg_all + (size_t)team * 2 * L * CC;  // x_s of the team in global memory, by parity
  double* xp = smem + cfg.xp;
  double* wv = smem + cfg.wv;
  double* prowb = smem + cfg.prow;
  double* apart = smem + cfg.apart;
  double* late = smem + cfg.late;
  double* rch = smem + cfg.rch;
  double* stages = smem + cfg.stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + cfg.bar);
  uint64_t* empty = full + S;
  const size_t stage_elems = (size_t)tpc * KC * 8;

  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, SWEEP_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // B operands start zeroed: padding columns read row CC, and a chunk's columns
  // past K multiply zero operand tiles, so those entries must be finite
  for (size_t i = tid; i < cfg.stage; i += SWEEP_THREADS_ALL) smem[i] = 0.0;
  __syncthreads();

  // ======================= producer warp: streams every job's A tiles =======================
  if (producer) {
    int jt = L, jph = 1;        // decode cursor (jobs with offsets)
    int ct = L, cph = 1;        // counting cursor (step boundaries)
    Job cur, nxt;
    bool has = false, has_nxt = false;
    int ch = 0, st = 0;
    long long issued = 0, target = 0;
    uint32_t ephase_bits = 0;   // per-stage parity of the next empty completion to wait for
    auto find_next = [&](Job& out) -> bool {
      int type, s;
      while (next_job_id(L, jt, jph, type, s)) {
        out = make_job(type, s, L, T, rank, SWEEP_KC, xt, xt_off, pbt, pb_off, true);
        if (out.nch > 0) return true;
      }
      return false;
    };
    auto count_step_chunks = [&](int steps) {  // advance the counting cursor over `steps` steps
      // prologue = BULK(L-1) only (ct = L, cph = 1); each later step t = CORR(t+1), BULK(t-1)
      for (int q = 0; q < steps; ++q) {
        int type, s;
        const int t_before = ct;
        while (ct == t_before && next_job_id(L, ct, cph, type, s))
          target += make_job(type, s, L, T, rank, SWEEP_KC, xt, xt_off, pbt, pb_off, false).nch;
      }
    };
    if (lane == 0) {
      has = find_next(cur);
      if (has) has_nxt = find_next(nxt);
    }
    auto pump = [&]() {  // issue until `target + S` chunks are out (blocking only on stages freed this step)
      if (lane != 0) return;
      while (has && issued < target + S) {
        if (issued >= S) {  // stage reuse: wait until every consumer warp released it
          mbar_wait(empty + st, (ephase_bits >> st) & 1u);
          ephase_bits ^= 1u << st;
        }
        uint64_t* bar = full + st;
        const uint32_t bytes = (uint32_t)((cur.rt1 - cur.rt0) * KC * 64);
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s(stages + st * stage_elems, cur.A + cur.off + ch * cur.cstride, bytes, bar);
        ++issued;
        if (++st == S) st = 0;
        if (++ch == cur.nch) {
          cur = nxt;
          has = has_nxt;
          ch = 0;
          if (has) has_nxt = find_next(nxt);
        }
      }
    };
    count_step_chunks(1);  // prologue: BULK(L-1)
    pump();
    __syncwarp();
    cluster.sync();
    for (int t = L - 1; t >= 0; --t) {
      count_step_chunks(1);
      pump();
      __syncwarp();
      cluster.sync();
    }
    return;
  }

  // ======================= consumer warps =======================
  PROF_DECL
  int cst = 0;          // stage of the next chunk to consume
  uint32_t cphase = 0;  // its full-barrier parity
  // Warp w owns output tiles w, w+8, ... (8 rows x 8 columns) of the job.
  auto run_job = [&](const Job& j, const double* Bsrc, int ldb, auto emit) {
    if (j.nch == 0) return;
    const int ntile = j.rt1 - j.rt0;
    const int items = ntile * NCT;
    int nmine = 0;
    int aoff[SWEEP_IPW], boff[SWEEP_IPW];
#pragma unroll
    for (int u = 0; u < SWEEP_IPW; ++u) {
      const int it = warp + u * SWEEP_WARPS;
      const bool ok = it < items;
      nmine += ok ? 1 : 0;
      const int rtl = ok ? it % ntile : 0, ct = ok ? it / ntile : 0;
      aoff[u] = rtl * SWEEP_KC * 8 + g;
      const int col = ct * 8 + g;
      boff[u] = ok && col < CC ? col : CC;  // column CC of Bsrc is a zero column
    }
    double res[SWEEP_IPW][2];
    switch (nmine) {
      case 1: job_tiles<1, CC>(j.nch, ldb, stages, stage_elems, full, empty, S, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
      case 2: job_tiles<2, CC>(j.nch, ldb, stages, stage_elems, full, empty, S, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
      case 3: job_tiles<3, CC>(j.nch, ldb, stages, stage_elems, full, empty, S, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
      case 4: job_tiles<4, CC>(j.nch, ldb, stages, stage_elems, full, empty, S, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
      default: {  // idle warp: keep the stage/phase bookkeeping and release the stages
        for (int ch = 0; ch < j.nch; ++ch) {
          mbar_wait(full + cst, cphase);
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + cst);
          if (++cst == S) {
            cst = 0;
            cphase ^= 1u;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < SWEEP_IPW; ++u) {
      if (u < nmine) {
        const int it = warp + u * SWEEP_WARPS;
        const int rtl = it % ntile, ct = it / ntile;
        const int c = ct * 8 + 2 * tq;
        if (c < CC) emit(8 * (j.rt0 + rtl) + g, c, res[u][0], res[u][1]);
      }
    }
  };

  // ---- gathered right-hand side of order s -> gst (row-major [j][ccp]) by cp.async
  int pidx[SWEEP_UMAX];
  auto load_perm = [&](int s) {  // data independent: one step ahead
    const int ns = L - s;
    const int* perm = perm_all + packed_pos(L, s, 0);
#pragma unroll
    for (int u = 0; u < SWEEP_UMAX; ++u) {
      const int jj = (tid + u * SWEEP_THREADS) / NB4;
      pidx[u] = (jj < ns) ? __ldg(perm + jj) : -1;
    }
  };
  auto gather_issue = [&](int s) {
    const int64_t ps = packed_pos(L, s, 0);
#pragma unroll
    for (int u = 0; u < SWEEP_UMAX; ++u) {
      const int idx = tid + u * SWEEP_THREADS;
      const int jj = idx / NB4, bl = idx % NB4;
      if (pidx[u] < 0) continue;
      double* dst = gst + (size_t)jj * ccp + 4 * bl;
      if (pidx[u] > 0 && bl < gm) {
        const int64_t base = ((ps + pidx[u]) * 2) * B + b0 + bl;
        cp_async16(dst, R + base);
        cp_async16(dst + 2, R + base + B);
      } else {  // late entry (ring s) is excluded from x'_s; padding map slots are zero
        dst[0] = dst[1] = dst[2] = dst[3] = 0.0;
      }
    }
  };
  // ---- x_s of the whole team (written to xg by its owners last step) -> xrow
  auto x_issue = [&](int s) {
    const int ns = L - s;
    const double* src = xg + (size_t)(s & 1) * L * CC;
    for (int idx = tid; idx < ns * (CC / 2); idx += SWEEP_THREADS) {
      const int l = idx / (CC / 2), c = 2 * (idx % (CC / 2));
      cp_async16(xrow + (size_t)l * ccp + c, src + (size_t)l * CC + c);
    }
  };
  auto load_rch = [&](int s) {  // R(+-)[s][0] of every map -> rch[s & 1] (synchronous)
    if (tid < gm) {
      const int64_t base = (packed_pos(L, s, 0) * 2) * B + b0 + tid;
      const double2 rp = __ldcg(R + base), rn = __ldcg(R + base + B);
      double* d = rch + (size_t)(s & 1) * CC + 4 * tid;
      d[0] = rp.x;
      d[1] = rp.y;
      d[2] = rn.x;
      d[3] = rn.y;
    }
  };
  auto rch_issue = [&](int s) {  // the same by cp.async (slots gm..NB4-1 stay zero)
    if (tid < gm) {
      const int64_t base = (packed_pos(L, s, 0) * 2) * B + b0 + tid;
      double* d = rch + (size_t)(s & 1) * CC + 4 * tid;
      cp_async16(d, R + base);
      cp_async16(d + 2, R + base + B);
    }
  };
  // data-independent operands of BULK(s) -> smem: w_s = X_s[own rows, j*_s] and
  // Pb_s[s-1, own rows]; the scalars (offsets, j*) are loaded one step earlier
  int64_t sx_off = 0, sp_off = 0;
  int sjs = 0;
  auto side_scalars = [&](int s) {
    if (s >= 0) {
      sx_off = __ldg(xt_off + s);
      sp_off = __ldg(pb_off + s);
      sjs = __ldg(jstar_all + s);
    }
  };
  auto side_issue = [&](int s) {
    const int ns = L - s, nrt = (ns + 7) / 8;
    const int r0 = 8 * ((rank * nrt) / T), r1 = min(ns, 8 * (((rank + 1) * nrt) / T));
    if (tid < r1 - r0) {
      const int l = r0 + tid;
      cp_async8(wv + (size_t)(s & 1) * ldr + tid, xt + sx_off + tile_index(l, sjs, nrt));
      if (s >= 1) cp_async8(prowb + tid, pbt + sp_off + tile_index(s - 1, l, (s + 7) >> 3));
    }
  };

  // BULK(s): x'_s on own rows, chain partial a_{s-1} (w_s and the Pb row are in
  // smem already).  The gathered right-hand side is unsigned; the (-1)^s of the
  // -m columns is applied here.
  auto bulk = [&](int s) {
    const Job j = make_job(0, s, L, T, rank, SWEEP_KC, xt, xt_off, pbt, pb_off, false);
    const int ns = j.K;
    const int r0 = 8 * j.rt0, r1 = min(ns, 8 * j.rt1);
    double* xps = xp + (size_t)(s & 1) * CC * ldr;
    const double ss = (s & 1) ? -1.0 : 1.0;
    run_job(j, gst, ccp, [&](int l, int c, double v0, double v1) {
      if (l < ns) {
        const double sg = (c & 2) ? ss : 1.0;
        xps[(size_t)c * ldr + (l - r0)] = sg * v0;
        xps[(size_t)(c + 1) * ldr + (l - r0)] = sg * v1;
      }
    });
    consumers_sync();
    PROF_MARK(6);
    if (s >= 1) {
      for (int c = warp; c < CC; c += SWEEP_WARPS) {
        double acc = 0.0;
        for (int l = lane; l < r1 - r0; l += 32) acc += prowb[l] * xps[(size_t)c * ldr + l];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane < T) *cluster.map_shared_rank(apart + ((s - 1) & 3) * T * CC + rank * CC + c, lane) = acc;
      }
    }
  };

  // ---- prologue: x'_{L-1}, a_{L-2}, R[L-1][0]
  load_perm(L - 1);
  side_scalars(L - 1);
  gather_issue(L - 1);
  side_issue(L - 1);
  cp_async_commit();
  cp_async_wait_all();
  consumers_sync();
  bulk(L - 1);
  load_rch(L - 1);
  if (L >= 2) load_perm(L - 2);
  side_scalars(L - 2);
  cluster.sync();

  double beta_next = L >= 2 ? __ldg(beta_all + L - 1) : 0.0;  // beta_{t+1} of the coming step
  for (int t = L - 1; t >= 0; --t) {
    const int nt = L - t;
    const double st = (t & 1) ? -1.0 : 1.0;
    const double bt = beta_next;
    const bool corr = t >= 1 && t + 1 <= L - 1;
    if (t >= 1) beta_next = __ldg(beta_all + t);  // consumed one step later
    // x_{t+1} (complete since the last cluster barrier) for CORR(t+1): group 1
    if (corr) x_issue(t + 1);
    cp_async_commit();
    // group 2: the right-hand side of order t-1 (final now: every correction but
    // the chain's has landed), its late entry R[t-1][0] and BULK(t-1)'s side operands
    if (t >= 1) {
      gather_issue(t - 1);
      side_issue(t - 1);
      if (t >= 2) rch_issue(t - 1);  // R[0][0] takes order-2 corrections at step 1
    }
    cp_async_commit();
    if (t >= 2) side_scalars(t - 2);
    if (t == 0) load_rch(0);
    PROF_MARK(0);
    // ---- (a) chain: late entries L_t of every map (threads tid < gm own map tid;
    // rch and late were written by the same threads)
    if (tid < NB4 && tid < gm) {
      const int b = tid;
      double gp_r = 0.0, gp_i = 0.0, gm_r = 0.0, gm_i = 0.0;  // G+_{t+1}(theta_t), G-_{t+1}(theta_t)
      if (t < L - 1) {
        const double s1 = ((t + 1) & 1) ? -1.0 : 1.0;
        double a[4] = {0.0, 0.0, 0.0, 0.0};
        const double* ap = apart + (size_t)(t & 3) * T * CC + 4 * b;
        for (int q = 0; q < T; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u) a[u] += ap[(size_t)q * CC + u];
        const double* ln = late + (size_t)((t + 1) & 1) * CC + 4 * b;
        gp_r = a[0] + bt * ln[0];
        gp_i = a[1] + bt * ln[1];
        gm_r = s1 * (a[2] + bt * ln[2]);
        gm_i = s1 * (a[3] + bt * ln[3]);
      }
      const double* rr = rch + (size_t)(t & 1) * CC + 4 * b;
      double* lt = late + (size_t)(t & 1) * CC + 4 * b;
      if (t == 0) {
        lt[0] = rr[0] - gp_r - gm_r;
        lt[1] = rr[1] - gp_i - gm_i;
        lt[2] = 0.0;
        lt[3] = 0.0;
      } else {
        lt[0] = rr[0] - gm_r;
        lt[1] = rr[1] - gm_i;
        lt[2] = st * (rr[2] - gp_r);
        lt[3] = st * (rr[3] - gp_i);
      }
    }
    consumers_sync();
    PROF_MARK(1);
    // ---- (b) x_t = x'_t + w_t L_t on own rows -> flm and the team exchange xg
    {
      const int nrt = (nt + 7) / 8;
      const int r0 = 8 * ((rank * nrt) / T), r1 = min(nt, 8 * (((rank + 1) * nrt) / T));
      const double* xps = xp + (size_t)(t & 1) * CC * ldr;
      const double* wvs = wv + (size_t)(t & 1) * ldr;
      const double* lt = late + (size_t)(t & 1) * CC;
      double* xo = xg + (size_t)(t & 1) * L * CC;
      for (int idx = tid; idx < (r1 - r0) * (CC / 2); idx += SWEEP_THREADS) {
        const int l = r0 + idx / (CC / 2), c = 2 * (idx % (CC / 2));
        const double wl = wvs[l - r0];
        const double v0 = xps[(size_t)c * ldr + (l - r0)] + wl * lt[c];
        const double v1 = xps[(size_t)(c + 1) * ldr + (l - r0)] + wl * lt[c + 1];
        __stcg(reinterpret_cast<double2*>(xo + (size_t)l * CC + c), make_double2(v0, v1));
        const int bl = c >> 2;
        if (bl < gm) {
          const int64_t ell = t + l;
          double2* f = flm + (int64_t)(b0 + bl) * L * L + ell * ell + ell;
          if ((c & 2) == 0) f[t] = make_double2(v0, v1);
          else if (t > 0) f[-t] = make_double2(v0, v1);
        }
      }
    }
    PROF_MARK(2);
    // ---- (c) CORR(t+1): corrections of order s = t+1 on own rings k < t
    if (corr) {
      const int s = t + 1;
      const double ss = (s & 1) ? -1.0 : 1.0;
      cp_async_wait_group1();
      consumers_sync();
      PROF_MARK(3);
      const Job j = make_job(1, s, L, T, rank, SWEEP_KC, xt, xt_off, pbt, pb_off, false);
      run_job(j, xrow, ccp, [&](int k, int c, double v0, double v1) {
        const int bl = c >> 2;
        if (k >= s - 1 || bl >= gm) return;  // ring s-1 is the chain
        const bool plus = (c & 2) == 0;
        const double gr = plus ? v0 : ss * v0, gi = plus ? v1 : ss * v1;
        const int nk = 2 * k + 1;
        const int r = s % nk;
        int tm, slot;
        if (r == 0) {
          tm = 0;
          slot = 0;
        } else if (r <= k) {
          tm = r;
          slot = plus ? 0 : 1;
        } else {
          tm = nk - r;
          slot = plus ? 1 : 0;
        }
        // fire-and-forget reductions (RED.ADD.F64): no load latency on the step's
        // critical path; at most two tones (r == 0) hit one bin per step
        double2* rp = R + (packed_pos(L, tm, k - tm) * 2 + slot) * B + b0 + bl;
        atomicAdd(&rp->x, -gr);
        atomicAdd(&rp->y, -gi);
      });
    }
    PROF_MARK(4);
    // ---- (d) BULK(t-1): x'_{t-1}, a_{t-2}; the next permutation
    if (t >= 1) {
      cp_async_wait_all();
      if (t >= 2) load_perm(t - 2);
      consumers_sync();
      PROF_MARK(5);
      bulk(t - 1);
    }
    PROF_MARK(7);
    cluster.sync();
    PROF_MARK(8);
  }
  PROF_DUMP();
}

static size_t sweep_smem_bytes(const SweepCfg& c) { return sizeof(double) * c.total; }

template <int CC>
static cudaError_t launch_sweep_cc(osph_plan* p, int B, int g, int T, int KC, int S, double2* flm) {
  const int L = p->L;
  const int teams = (B + g - 1) / g;
  const SweepCfg cfg(L, T, CC, KC, S);
  const size_t smem = sweep_smem_bytes(cfg);
  auto kern = k_sweep<CC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (T > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
    return e;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(teams * T));
  lc.blockDim = dim3(SWEEP_THREADS_ALL);
  lc.dynamicSmemBytes = smem;
  lc.stream = p->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = T;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  if (getenv("OSPH_DEBUG")) {
    int nclusters = -1;
    cudaOccupancyMaxActiveClusters(&nclusters, (void*)kern, &lc);
    fprintf(stderr, "[osph] sweep L=%d B=%d maps/team=%d teams=%d T=%d KC=%d S=%d smem=%zu maxActiveClusters=%d\n", L,
            B, g, teams, T, KC, S, smem, nclusters);
  }
  e = cudaLaunchKernelEx(&lc, kern, L, B, g, KC, S, (const double*)p->d_xt, (const int64_t*)p->d_xt_off,
                         (const int*)p->d_piv, (const int*)p->d_jstar, (const double*)p->d_beta,
                         (const double*)p->d_pbelow, (const int64_t*)p->d_pb_off, p->d_r, flm, p->d_xg);
  p->launches++;
  return e;
}

template <int CC>
static int max_active_clusters(int L, int T, int KC, int S) {
  const size_t smem = sweep_smem_bytes(SweepCfg(L, T, CC, KC, S));
  auto kern = k_sweep<CC>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  if (T > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)T);
  lc.blockDim = dim3(SWEEP_THREADS_ALL);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = T;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void*)kern, &lc) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

cudaError_t launch_sweep(osph_plan* p, int B, double2* flm) {
  const int L = p->L;
  const size_t cap = 220 * 1024;
  const int KC = SWEEP_KC;
  if (p->sweep_cfg_B == B && !getenv("OSPH_SWEEP_T") && !getenv("OSPH_SWEEP_G") && !getenv("OSPH_SWEEP_S")) {
    const int g = p->sweep_cfg[0], T = p->sweep_cfg[1], S = p->sweep_cfg[2];
    if (g == 4) return launch_sweep_cc<16>(p, B, 4, T, KC, S, flm);
    if (g == 2) return launch_sweep_cc<8>(p, B, 2, T, KC, S, flm);
    return launch_sweep_cc<4>(p, B, 1, T, KC, S, flm);
  }
  // maps per team: 4 (16 columns) / 2 / 1, limited by the register-held
  // gather (L * CC/4 <= 8 * 256) and by shared memory
  int g = B >= 3 ? 4 : B;
  while (g > 1 && (size_t)L * g > (size_t)SWEEP_UMAX * SWEEP_THREADS) g /= 2;
  g = std::min(g, std::max(1, env_int("OSPH_SWEEP_G", g)));
  // a job's tiles must fit one row of threads (side loads) and the per-warp accumulators
  auto tiles_ok = [&](int gg, int TT) {
    const int tpc = ((L + 7) / 8 + TT - 1) / TT;
    return tpc <= 32 && tpc * ((4 * gg + 7) / 8) <= SWEEP_WARPS * SWEEP_IPW;
  };
  auto fits = [&](int gg, int TT, int ss) { return sweep_smem_bytes(SweepCfg(L, TT, 4 * gg, KC, ss)) <= cap; };
  auto mac = [&](int gg, int TT, int ss) {
    return gg == 4 ? max_active_clusters<16>(L, TT, KC, ss)
                   : gg == 2 ? max_active_clusters<8>(L, TT, KC, ss) : max_active_clusters<4>(L, TT, KC, ss);
  };
  // Largest team (cluster) width T whose configuration fits shared memory and
  // keeps every team resident at once (teams never wait on each other, but a
  // second wave doubles the latency-bound wall time); deepest ring that fits.
  // Over maps-per-team g (<= the register limit above) and T, maximise the CTAs
  // at work subject to residency; ties go to more maps per team (less L2 traffic).
  int T = 1, S = 3, best_ctas = 0, best_g = g;
  bool found = false;
  const int gmax = g;
  for (int gg = gmax; gg >= 1; gg /= 2) {
    const int teams = (B + gg - 1) / gg;
    for (int TT = 16; TT >= 1; TT /= 2) {
      if (TT * 32 > 2 * L && TT > 1) continue;  // a team wider than the rows is idle
      if (!tiles_ok(gg, TT)) continue;
      int ss = SWEEP_SMAX;
      while (ss >= 3 && !fits(gg, TT, ss)) --ss;
      if (ss < 3) continue;
      if (mac(gg, TT, ss) < teams) continue;
      if (teams * TT > best_ctas) {
        best_ctas = teams * TT;
        best_g = gg;
        T = TT;
        S = ss;
        found = true;
      }
      break;  // narrower teams of this g only lose CTAs
    }
    if (gg == 1) break;
  }
  if (found) g = best_g;
  if (!found) {  // several waves of teams: take the narrowest team that fits
    for (int TT = 1; TT <= 16; TT *= 2)
      if (tiles_ok(g, TT) && fits(g, TT, 3)) {
        T = TT;
        break;
      }
    S = 3;
    while (S < SWEEP_SMAX && fits(g, T, S + 1)) ++S;
  }
  T = env_int("OSPH_SWEEP_T", T);
  S = env_int("OSPH_SWEEP_S", S);
  p->sweep_cfg_B = B;
  p->sweep_cfg[0] = g;
  p->sweep_cfg[1] = T;
  p->sweep_cfg[2] = S;
  if (g == 4) return launch_sweep_cc<16>(p, B, 4, T, KC, S, flm);
  if (g == 2) return launch_sweep_cc<8>(p, B, 2, T, KC, S, flm);
  return launch_sweep_cc<4>(p, B, 1, T, KC, S, flm);
}
