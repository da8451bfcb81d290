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
// cluster barrier.  Step t (t = L-1 .. 0) has three independent tasks:
//   chain/CORR warps:  (a) chain -> L_t; (b) x_t = x'_t + w_t L_t on own rows
//                      -> flm and the team exchange buffer; (c) CORR(t+1):
//                      corrections of order t+1 (x_{t+1} complete) on own rings
//   BULK warps:        (d) BULK(t-1): x'_{t-1} on own rows, chain partial
//                      a_{t-2} -> DSMEM
// and the two warp groups run them concurrently, so a step costs the longer of
// the two paths plus one barrier instead of their sum.  x'_s is computed one
// step before it is used; the corrections of order s+1 are applied one step
// after x_{s+1} is known -- both fit the alias dependency structure (orders
// >= s+3 feed the non-late entries of order s).
//
// Streaming.  CORR and BULK are row-sliced GEMMs (rows of the team split
// over its CTAs, K = n) on the fp64 tensor cores (mma.sync m8n8k4 ->
// DMMA.8x8x4).  Their A operands (8-row tiles of Pb_s / X_s, written by the
// factorisation) do not depend on the data, so one producer warp per group
// streams them with bulk async copies (cp.async.bulk + mbarrier complete_tx,
// the TMA engine) through an S-stage ring that runs ahead across steps; only
// the small B operands (x, gathered right-hand sides) wait on the chain.
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

#define SWEEP_WC 4      // chain/CORR warps
#define SWEEP_WB 4      // BULK warps
#define SWEEP_NC (SWEEP_WC * 32)
#define SWEEP_NB (SWEEP_WB * 32)
#define SWEEP_THREADS_ALL (SWEEP_NC + SWEEP_NB + 64)  // + one producer warp per group
#define SWEEP_IPW 4     // max accumulator tiles per warp
#define SWEEP_KC 32     // K columns per streamed chunk
#define SWEEP_SMAX 6    // ring stages per group
#define SWEEP_BAR_C 1   // named barriers of the two groups
#define SWEEP_BAR_B 2

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
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
// full cluster barrier (release/acquire: orders the step's global, shared and
// DSMEM writes before every CTA's next step)
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// a mod n for 0 <= a < 2^22, 0 < n < 2^22 without an integer division
__device__ __forceinline__ int mod_small(int a, int n) {
  const int q = __float2int_rz(__fdividef((float)a, (float)n));
  int r = a - q * n;
  if (r < 0) r += n;
  if (r >= n) r -= n;
  return r;
}
// named barrier of one warp group (the other groups and the producers never join it)
__device__ __forceinline__ void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// -DOSPH_SWEEP_PROF: per-phase cycle counts of CTA 0, per warp group (debug builds only)
#ifdef OSPH_SWEEP_PROF
#define PROF_DECL            \
  long long _pt = clock64(); \
  long long _acc[6] = {};
#define PROF_MARK(i)                \
  do {                              \
    group_sync(gbar, gn);           \
    const long long _n = clock64(); \
    _acc[i] += _n - _pt;            \
    _pt = _n;                       \
  } while (0)
#define PROF_DUMP(name)                                                                                     \
  if (blockIdx.x == 0 && gt == 0)                                                                           \
  printf("sweep prof %s (cycles): %lld %lld %lld %lld %lld %lld\n", name, _acc[0], _acc[1], _acc[2], _acc[3], \
         _acc[4], _acc[5])
#else
#define PROF_DECL
#define PROF_MARK(i)
#define PROF_DUMP(name)
#endif

// ---------------------------------------------------------------------------
// configuration and shared-memory layout

struct SweepCfg {
  int L, T, CC, KC, S;
  int tpc;  // max 8-row tiles of one job on one CTA
  int ldx, ldr, ccp;
  size_t xrow, gst, xp, wv, ubuf, apart, late, rch, permb, stage, bar, total;  // offsets in doubles
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
    ubuf = o;  o += (size_t)ldx;                // u_s = Pb_s[s-1, :] X_s (chain partial weights)
    apart = o; o += (size_t)4 * CC;             // chain partials a_s, slot s % 4
    late = o;  o += (size_t)2 * CC;             // late right-hand-side entries L_s, by parity
    rch = o;   o += (size_t)2 * CC;             // prefetched R(+-)[s][0], by parity
    permb = o; o += (size_t)ldx;                // pivot order of order s (ints), by parity
    o = (o + 15) & ~(size_t)15;                 // 128-byte aligned stages
    stage = o; o += (size_t)2 * S * tpc * KC * 8;  // ring B (BULK) then ring C (CORR)
    bar = o;   o += (size_t)4 * S;              // fullB[S], emptyB[S], fullC[S], emptyC[S]
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

__device__ __forceinline__ Job make_job(int type, int s, int L, int lgT, int rank, int KC, const double* xt,
                                        const int64_t* xt_off, const double* pbt, const int64_t* pb_off,
                                        bool with_offset) {
  Job j;
  j.type = type;
  j.s = s;
  j.K = L - s;
  const int rows = type == 0 ? j.K : s - 1;  // CORR skips ring s-1 (the chain)
  const int mrows = type == 0 ? j.K : s;     // rows of the stored matrix
  const int nt = (rows + 7) / 8;
  j.rt0 = (rank * nt) >> lgT;  // team width T = 2^lgT
  j.rt1 = ((rank + 1) * nt) >> lgT;
  j.nch = (j.rt1 > j.rt0 && rows > 0) ? (j.K + KC - 1) / KC : 0;
  j.cstride = (int64_t)((mrows + 7) / 8) * KC * 8;
  j.A = type == 0 ? xt : pbt;
  j.off = with_offset ? (type == 0 ? xt_off[s] : pb_off[s]) + (int64_t)j.rt0 * KC * 8 : 0;
  return j;
}

// A streaming ring: S stages of `stage_elems` doubles with full/empty barriers.
struct Ring {
  double* stages;
  uint64_t* full;
  uint64_t* empty;
  size_t stage_elems;
  int S;
};

// One job's chunk loop for a warp owning NM output tiles (8x8 each), with
// CH independent accumulator chains per tile for DMMA latency hiding.
template <int NM>
__device__ __forceinline__ void job_tiles(int nch, int ldb, const Ring& rg, int& cst, uint32_t& cphase,
                                          const int* aoff, const int* boff, const double* Bsrc, int tq, int lane,
                                          double (&out)[SWEEP_IPW][2]) {
  constexpr int CH = NM == 1 ? 8 : NM == 2 ? 4 : 2;  // independent chains per tile
  double acc[NM][CH][2];
#pragma unroll
  for (int u = 0; u < NM; ++u)
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[u][c][0] = acc[u][c][1] = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    mbar_wait(rg.full + cst, cphase);
    const double* sA = rg.stages + cst * rg.stage_elems + tq * 8;
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
    if (lane == 0) mbar_arrive(rg.empty + cst);
    if (++cst == rg.S) {
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

// Warp gw of a group of NW warps owns output tiles gw, gw+NW, ... (8 rows x 8
// columns) of the job; emit(row, column, v0, v1) gets two adjacent columns.
template <int CC, typename Emit>
__device__ __forceinline__ void run_job(const Job& j, const Ring& rg, int& cst, uint32_t& cphase, int gw, int NW,
                                        const double* Bsrc, int ldb, int g, int tq, int lane, Emit emit) {
  constexpr int NCT = (CC + 7) / 8;
  if (j.nch == 0) return;
  const int ntile = j.rt1 - j.rt0;
  const int items = ntile * NCT;
  int nmine = 0;
  int aoff[SWEEP_IPW], boff[SWEEP_IPW];
#pragma unroll
  for (int u = 0; u < SWEEP_IPW; ++u) {
    const int it = gw + u * NW;
    const bool ok = it < items;
    nmine += ok ? 1 : 0;
    const int ct = (NCT == 2 && it >= ntile) ? 1 : 0;  // NCT <= 2: no division
    const int rtl = ok ? it - ct * ntile : 0;
    aoff[u] = rtl * SWEEP_KC * 8 + g;
    const int col = ct * 8 + g;
    boff[u] = ok && col < CC ? col : CC;  // column CC of Bsrc is a zero column
  }
  double res[SWEEP_IPW][2];
  switch (nmine) {
    case 1: job_tiles<1>(j.nch, ldb, rg, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
    case 2: job_tiles<2>(j.nch, ldb, rg, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
    case 3: job_tiles<3>(j.nch, ldb, rg, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
    case 4: job_tiles<4>(j.nch, ldb, rg, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
    default: {  // idle warp: keep the stage/phase bookkeeping and release the stages
      for (int ch = 0; ch < j.nch; ++ch) {
        mbar_wait(rg.full + cst, cphase);
        __syncwarp();
        if (lane == 0) mbar_arrive(rg.empty + cst);
        if (++cst == rg.S) {
          cst = 0;
          cphase ^= 1u;
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < SWEEP_IPW; ++u) {
    if (u < nmine) {
      const int it = gw + u * NW;
      const int ct = (NCT == 2 && it >= ntile) ? 1 : 0;
      const int rtl = it - ct * ntile;
      const int c = ct * 8 + 2 * tq;
      if (c < CC) emit(8 * (j.rt0 + rtl) + g, c, res[u][0], res[u][1]);
    }
  }
}

// Producer of one ring (lane 0 of a producer warp).  The ring's jobs are
// consumed one per step in a fixed order; `step_job(q)` gives the job of step
// q (prologue = q 0) or type -1.  Per step the producer issues until the
// chunks of this step plus S more are out -- every stage it waits for is
// released within the current step, so the per-step cluster barrier cannot
// deadlock with a blocked producer.
template <typename StepJob>
__device__ __forceinline__ void produce(const Ring& rg, int nsteps, int lane,
                                        StepJob step_job) {
  Job cur;
  int q_dec = 0;  // next step whose job is decoded
  bool has = false;
  int ch = 0, st = 0;
  long long issued = 0, target = 0;
  uint32_t ephase_bits = 0;  // per-stage parity of the next empty completion to wait for
  auto next = [&]() {
    has = false;
    while (q_dec < nsteps) {
      cur = step_job(q_dec++, true);
      if (cur.type >= 0 && cur.nch > 0) {
        has = true;
        return;
      }
    }
  };
  if (lane == 0) next();
  for (int q = 0; q < nsteps; ++q) {
    if (lane == 0) {
      const Job jq = step_job(q, false);
      if (jq.type >= 0) target += jq.nch;
      while (has && issued < target + rg.S) {
        if (issued >= rg.S) {  // stage reuse: wait until every consumer warp released it
          mbar_wait(rg.empty + st, (ephase_bits >> st) & 1u);
          ephase_bits ^= 1u << st;
        }
        uint64_t* bar = rg.full + st;
        const uint32_t bytes = (uint32_t)((cur.rt1 - cur.rt0) * SWEEP_KC * 64);
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s(rg.stages + st * rg.stage_elems, cur.A + cur.off + ch * cur.cstride, bytes, bar);
        ++issued;
        if (++st == rg.S) st = 0;
        if (++ch == cur.nch) {
          ch = 0;
          next();
        }
      }
    }
    __syncwarp();
    cluster_sync_all();
  }
}

template <int CC>
__global__ void __launch_bounds__(SWEEP_THREADS_ALL, 1) k_sweep(
    int L, int B, int maps_per_team, int KC, int S, const double* __restrict__ xt, const int64_t* __restrict__ xt_off,
    const int* __restrict__ perm_all, const int* __restrict__ jstar_all, const double* __restrict__ beta_all,
    const double* __restrict__ pbt, const int64_t* __restrict__ pb_off, double2* __restrict__ R,
    double2* __restrict__ flm, double* __restrict__ xg_all, const double* __restrict__ u_all) {
  cg::cluster_group cluster = cg::this_cluster();
  const int T = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int lgT = __ffs(T) - 1;  // T is a power of two (launch_sweep)
  const int team = (int)(blockIdx.x >> lgT);
  const int b0 = team * maps_per_team;
  const int gm = min(maps_per_team, B - b0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  constexpr int NB4 = CC / 4;  // map slots of the team

  extern __shared__ __align__(128) double smem[];
  const SweepCfg cfg(L, T, CC, KC, S);
  const int ldr = cfg.ldr, tpc = cfg.tpc, ccp = cfg.ccp;
  double* xrow = smem + cfg.xrow;
  double* gst = smem + cfg.gst;
  double* xg = xg_all + (size_t)team * 2 * L * CC;  // x_s of the team in global memory, by parity
  double* xp = smem + cfg.xp;
  double* wv = smem + cfg.wv;
  double* ubuf = smem + cfg.ubuf;
  double* apart = smem + cfg.apart;
  double* late = smem + cfg.late;
  double* rch = smem + cfg.rch;
  int* permb = reinterpret_cast<int*>(smem + cfg.permb);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + cfg.bar);
  const size_t stage_elems = (size_t)tpc * KC * 8;
  const Ring ringB{smem + cfg.stage, bars, bars + S, stage_elems, S};
  const Ring ringC{smem + cfg.stage + (size_t)S * stage_elems, bars + 2 * S, bars + 3 * S, stage_elems, S};

  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(ringB.full + i, 1);
      mbar_init(ringB.empty + i, SWEEP_WB);
      mbar_init(ringC.full + i, 1);
      mbar_init(ringC.empty + i, SWEEP_WC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // B operands start zeroed: padding columns read column CC, and a chunk's
  // rows past K multiply zero operand tiles, so those entries must be finite
  for (size_t i = tid; i < cfg.stage; i += SWEEP_THREADS_ALL) smem[i] = 0.0;
  __syncthreads();

  // Steps: q = 0 is the prologue, q = L - t is step t.
  const int nsteps = L + 1;

  // ======================= producers =======================
  if (warp == SWEEP_WC + SWEEP_WB) {  // ring B: BULK(L-1) in the prologue, BULK(t-1) at step t
    produce(ringB, nsteps, lane, [&](int q, bool off) {
      const int s = L - 1 - q;  // q = 0 -> L-1; step t (q = L-t) -> t-1
      Job j;
      if (s < 0) {
        j.type = -1;
        return j;
      }
      return make_job(0, s, L, lgT, rank, SWEEP_KC, xt, xt_off, pbt, pb_off, off);
    });
    return;
  }
  if (warp == SWEEP_WC + SWEEP_WB + 1) {  // ring C: CORR(t+1) at step t, 1 <= t <= L-2
    produce(ringC, nsteps, lane, [&](int q, bool off) {
      const int t = L - q;
      Job j;
      if (q == 0 || t < 1 || t > L - 2) {
        j.type = -1;
        return j;
      }
      return make_job(1, t + 1, L, lgT, rank, SWEEP_KC, xt, xt_off, pbt, pb_off, off);
    });
    return;
  }

  if (warp < SWEEP_WC) {
    // ======================= chain / CORR warps =======================
    const int gt = tid, gw = warp;
    const int gbar = SWEEP_BAR_C, gn = SWEEP_NC;
    (void)gbar;
    (void)gn;
    PROF_DECL
    int cst = 0;
    uint32_t cphase = 0;
    auto load_rch = [&](int s) {  // R(+-)[s][0] of every map -> rch[s & 1] (synchronous)
      if (gt < gm) {
        const int64_t base = (packed_pos(L, s, 0) * 2) * B + b0 + gt;
        const double2 rp = __ldcg(R + base), rn = __ldcg(R + base + B);
        double* d = rch + (size_t)(s & 1) * CC + 4 * gt;
        d[0] = rp.x;
        d[1] = rp.y;
        d[2] = rn.x;
        d[3] = rn.y;
      }
    };
    auto rch_issue = [&](int s) {  // the same by cp.async (slots gm..NB4-1 stay zero)
      if (gt < gm) {
        const int64_t base = (packed_pos(L, s, 0) * 2) * B + b0 + gt;
        double* d = rch + (size_t)(s & 1) * CC + 4 * gt;
        cp_async16(d, R + base);
        cp_async16(d + 2, R + base + B);
      }
    };
    load_rch(L - 1);
    cluster_sync_all();  // prologue
    double beta_next = L >= 2 ? __ldg(beta_all + L - 1) : 0.0;  // beta_{t+1} of the coming step
    for (int t = L - 1; t >= 0; --t) {
      const int nt = L - t;
      const double st = (t & 1) ? -1.0 : 1.0;
      const double bt = beta_next;
      const bool corr = t >= 1 && t + 1 <= L - 1;
      if (t >= 1) beta_next = __ldg(beta_all + t);  // consumed one step later
      // x_{t+1} (complete since the last cluster barrier) for CORR(t+1), and the
      // late entry R[t-1][0] of the next step (final now; R[0][0] takes order-2
      // corrections at step 1 and is read synchronously at step 0)
      if (corr) {
        const double* src = xg + (size_t)((t + 1) & 1) * L * CC;
        for (int idx = gt; idx < (nt - 1) * (CC / 2); idx += SWEEP_NC) {
          const int l = idx / (CC / 2), c = 2 * (idx % (CC / 2));
          cp_async16(xrow + (size_t)l * ccp + c, src + (size_t)l * CC + c);
        }
      }
      if (t >= 2) rch_issue(t - 1);
      cp_async_commit();
      if (t == 0) load_rch(0);
      PROF_MARK(0);
      // ---- (a) chain: late entries L_t of every map (threads gt < gm own map gt;
      // rch and late were written by the same threads)
      if (gt < gm) {
        const int b = gt;
        double gp_r = 0.0, gp_i = 0.0, gm_r = 0.0, gm_i = 0.0;  // G+_{t+1}(theta_t), G-_{t+1}(theta_t)
        if (t < L - 1) {
          const double s1 = ((t + 1) & 1) ? -1.0 : 1.0;
          const double* a = apart + (size_t)(t & 3) * CC + 4 * b;
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
      group_sync(SWEEP_BAR_C, SWEEP_NC);
      PROF_MARK(1);
      // ---- (b) x_t = x'_t + w_t L_t on own rows -> flm and the team exchange xg
      {
        const int nrt = (nt + 7) / 8;
        const int r0 = 8 * ((rank * nrt) >> lgT), r1 = min(nt, 8 * (((rank + 1) * nrt) >> lgT));
        const double* xps = xp + (size_t)(t & 1) * CC * ldr;
        const double* wvs = wv + (size_t)(t & 1) * ldr;
        const double* lt = late + (size_t)(t & 1) * CC;
        double* xo = xg + (size_t)(t & 1) * L * CC;
        for (int idx = gt; idx < (r1 - r0) * (CC / 2); idx += SWEEP_NC) {
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
      cp_async_wait_all();
      // ---- (c) CORR(t+1): corrections of order s = t+1 on own rings k < t
      if (corr) {
        const int s = t + 1;
        const double ss = (s & 1) ? -1.0 : 1.0;
        group_sync(SWEEP_BAR_C, SWEEP_NC);
        PROF_MARK(3);
        const Job j = make_job(1, s, L, lgT, rank, SWEEP_KC, xt, xt_off, pbt, pb_off, false);
        run_job<CC>(j, ringC, cst, cphase, gw, SWEEP_WC, xrow, ccp, g, tq, lane, [&](int k, int c, double v0, double v1) {
          const int bl = c >> 2;
          if (k >= s - 1 || bl >= gm) return;  // ring s-1 is the chain
          const bool plus = (c & 2) == 0;
          const double gr = plus ? v0 : ss * v0, gi = plus ? v1 : ss * v1;
          const int nk = 2 * k + 1;
          const int r = mod_small(s, nk);
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
      cluster_sync_all();
      PROF_MARK(5);
    }
    PROF_DUMP("chain/corr");
    return;
  }

  // ======================= BULK warps =======================
  {
    const int gt = tid - SWEEP_NC, gw = warp - SWEEP_WC;
    const int gbar = SWEEP_BAR_B, gn = SWEEP_NB;
    (void)gbar;
    (void)gn;
    PROF_DECL
    int cst = 0;
    uint32_t cphase = 0;
    // pivot order of order s -> permb[s & 1] (one step ahead, by cp.async)
    auto perm_issue = [&](int s) {
      const int ns = L - s;
      const int* perm = perm_all + packed_pos(L, s, 0);
      int* d = permb + (size_t)(s & 1) * cfg.ldx;
      for (int i = gt; i < ns; i += SWEEP_NB) cp_async4(d + i, perm + i);
    };
    // gathered right-hand side of order s -> gst (row-major [j][ccp]), unsigned
    auto gather_issue = [&](int s) {
      const int ns = L - s;
      const int64_t ps = packed_pos(L, s, 0);
      const int* pm = permb + (size_t)(s & 1) * cfg.ldx;
      for (int idx = gt; idx < ns * NB4; idx += SWEEP_NB) {
        const int jj = idx / NB4, bl = idx % NB4;
        const int pj = pm[jj];
        double* dst = gst + (size_t)jj * ccp + 4 * bl;
        if (pj > 0 && bl < gm) {
          const int64_t base = ((ps + pj) * 2) * B + b0 + bl;
          cp_async16(dst, R + base);
          cp_async16(dst + 2, R + base + B);
        } else {  // late entry (ring s) is excluded from x'_s; padding map slots are zero
          dst[0] = dst[1] = dst[2] = dst[3] = 0.0;
        }
      }
    };
    // data-independent operands of BULK(s) -> smem: w_s = X_s[own rows, j*_s] and
    // u_s; the scalars (offset, j*) are loaded one step earlier
    int64_t sx_off = 0;
    int sjs = 0;
    auto side_scalars = [&](int s) {
      if (s >= 0) {
        sx_off = __ldg(xt_off + s);
        sjs = __ldg(jstar_all + s);
      }
    };
    auto side_issue = [&](int s) {
      const int ns = L - s, nrt = (ns + 7) / 8;
      const int r0 = 8 * ((rank * nrt) >> lgT), r1 = min(ns, 8 * (((rank + 1) * nrt) >> lgT));
      for (int i = gt; i < r1 - r0; i += SWEEP_NB)
        cp_async8(wv + (size_t)(s & 1) * ldr + i, xt + sx_off + tile_index(r0 + i, sjs, nrt));
      if (s >= 1) {
        const double* us = u_all + packed_pos(L, s, 0);
        for (int i = gt; i < ns; i += SWEEP_NB) cp_async8(ubuf + i, us + i);
      }
    };
    // BULK(s): x'_s on own rows (the (-1)^s of the -m columns applied here),
    // and the chain partial a_{s-1} = u_s . (P rhs_s) of the whole team: every
    // CTA holds the full gathered right-hand side, so no exchange is needed
    auto bulk = [&](int s) {
      const Job j = make_job(0, s, L, lgT, rank, SWEEP_KC, xt, xt_off, pbt, pb_off, false);
      const int ns = j.K;
      const int r0 = 8 * j.rt0;
      double* xps = xp + (size_t)(s & 1) * CC * ldr;
      const double ss = (s & 1) ? -1.0 : 1.0;
      run_job<CC>(j, ringB, cst, cphase, gw, SWEEP_WB, gst, ccp, g, tq, lane, [&](int l, int c, double v0, double v1) {
        if (l < ns) {
          const double sg = (c & 2) ? ss : 1.0;
          xps[(size_t)c * ldr + (l - r0)] = sg * v0;
          xps[(size_t)(c + 1) * ldr + (l - r0)] = sg * v1;
        }
      });
      PROF_MARK(3);
      if (s >= 1) {
        for (int c = gw; c < CC; c += SWEEP_WB) {
          double acc = 0.0;
          for (int l = lane; l < ns; l += 32) acc += ubuf[l] * gst[(size_t)l * ccp + c];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (lane == 0) apart[((s - 1) & 3) * CC + c] = (c & 2) ? ss * acc : acc;
        }
      }
    };

    // ---- prologue: x'_{L-1}, a_{L-2}
    perm_issue(L - 1);
    side_scalars(L - 1);
    cp_async_commit();
    cp_async_wait_all();
    group_sync(SWEEP_BAR_B, SWEEP_NB);
    gather_issue(L - 1);
    side_issue(L - 1);
    if (L >= 2) perm_issue(L - 2);
    cp_async_commit();
    cp_async_wait_all();
    group_sync(SWEEP_BAR_B, SWEEP_NB);
    bulk(L - 1);
    side_scalars(L - 2);
    cluster_sync_all();
    for (int t = L - 1; t >= 0; --t) {
      if (t >= 1) {
        // the right-hand side of order t-1 is final now: every correction but
        // the chain's has landed
        gather_issue(t - 1);
        side_issue(t - 1);
        if (t >= 2) perm_issue(t - 2);
        cp_async_commit();
        if (t >= 2) side_scalars(t - 2);
        PROF_MARK(0);
        cp_async_wait_all();
        group_sync(SWEEP_BAR_B, SWEEP_NB);
        PROF_MARK(1);
        bulk(t - 1);
      }
      PROF_MARK(4);
      cluster_sync_all();
      PROF_MARK(5);
    }
    PROF_DUMP("bulk");
  }
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
                         (const double*)p->d_pbelow, (const int64_t*)p->d_pb_off, p->d_r, flm, p->d_xg, (const double*)p->d_u);
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
  // maps per team: 4 (16 columns) / 2 / 1, limited by shared memory
  int g = B >= 3 ? 4 : B;
  g = std::min(g, std::max(1, env_int("OSPH_SWEEP_G", g)));
  // a job's tiles must fit one row of threads (side loads) and the per-warp accumulators
  auto tiles_ok = [&](int gg, int TT) {
    const int tpc = ((L + 7) / 8 + TT - 1) / TT;
    return tpc <= 32 && tpc * ((4 * gg + 7) / 8) <= std::min(SWEEP_WB, SWEEP_WC) * SWEEP_IPW;
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
  while (T & (T - 1)) T &= T - 1;  // the kernel needs a power-of-two team width
  S = env_int("OSPH_SWEEP_S", S);
  p->sweep_cfg_B = B;
  p->sweep_cfg[0] = g;
  p->sweep_cfg[1] = T;
  p->sweep_cfg[2] = S;
  if (g == 4) return launch_sweep_cc<16>(p, B, 4, T, KC, S, flm);
  if (g == 2) return launch_sweep_cc<8>(p, B, 2, T, KC, S, flm);
  return launch_sweep_cc<4>(p, B, 1, T, KC, S, flm);
}
