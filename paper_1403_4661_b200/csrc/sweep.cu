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
#define SWEEP_THREADS_ALL (SWEEP_NC + SWEEP_NB + 96)  // + one producer warp per group + the output warp
#define SWEEP_IPW 4     // max accumulator tiles per warp
#define SWEEP_KC 32     // K columns per streamed chunk
#define SWEEP_SMAX 6    // ring stages per group
#define SWEEP_BAR_C 1   // named barriers of the two groups
#define SWEEP_BAR_B 2
#define SWEEP_PF_MIN 2  // orders >= this get their right-hand side prefetched a step early

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
#ifdef OSPH_SWEEP_PROF
__device__ long long g_prof_arrive[16];  // per warp of CTA 0: cycles spent inside the release arrive
#endif
// Step barrier.  MODE 0: release arrival (MEMBAR.GPU + ERRBAR: waits for every
// outstanding write of the warp); 1: CTA-scope fence + relaxed arrival (the
// warp's writes are only read inside its own CTA); 2: relaxed arrival (no
// writes to order, or ordered by an earlier explicit fence).  Always an
// acquire wait.
template <int MODE>
__device__ __forceinline__ void step_barrier() {
#ifdef OSPH_SWEEP_PROF
  const long long ta = clock64();
#endif
  if (MODE == 0) asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  if (MODE == 1) asm volatile("fence.acq_rel.cta;\nbarrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  if (MODE == 2) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
#ifdef OSPH_SWEEP_PROF
  const long long tb = clock64();
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) g_prof_arrive[threadIdx.x >> 5] += tb - ta;
#endif
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_all() { step_barrier<0>(); }
// Alias target of a correction of order s on ring k: R[pos(tm, k - tm)][slot]
// (transform.py:459-463 in the order-major layout).  r == 0 puts both tones in
// bin 0 (order 0): the + tone into its + slot, the - tone into order 0's unused
// - slot (zeroed by the ring DFT scatter), so the two reductions never race on
// one address (bitwise-reproducible sums); the slots are added before order 0
// is solved.
__device__ __forceinline__ int mod_small(int a, int n);
__device__ __forceinline__ void corr_target(int s, int k, bool plus, int& tm, int& slot) {
  const int nk = 2 * k + 1;
  const int r = mod_small(s, nk);
  if (r == 0) {
    tm = 0;
    slot = plus ? 0 : 1;
  } else if (r <= k) {
    tm = r;
    slot = plus ? 0 : 1;
  } else {
    tm = nk - r;
    slot = plus ? 1 : 0;
  }
}
// a mod n for 0 <= a < 2^22, 0 < n < 2^22 without an integer division
__device__ __forceinline__ int mod_small(int a, int n) {
  const int q = __float2int_rz(__fdividef((float)a, (float)n));
  int r = a - q * n;
  if (r < 0) r += n;
  if (r >= n) r -= n;
  return r;
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// shared::cluster address of `p` (a local shared-memory pointer) in CTA `rank`
__device__ __forceinline__ uint32_t mapa_u32(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// generic-proxy accesses before async-proxy (bulk copy) accesses of the same memory
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;\n" ::: "memory"); }
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
  if (blockIdx.x < 4 && gt == 0)                                                                            \
  printf("sweep prof %s cta %d (cycles): %lld %lld %lld %lld %lld %lld\n", name, (int)blockIdx.x, _acc[0], _acc[1], _acc[2], _acc[3], \
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
  int ldx, ldr;
  size_t gst, xrow, xst, xp, wv, ubuf, fix, apart, late, rch, stage, bar, total;  // offsets in doubles
  __host__ __device__ SweepCfg(int L_, int T_, int CC_, int KC_, int S_) : L(L_), T(T_), CC(CC_), KC(KC_), S(S_) {
    tpc = ((L + 7) / 8 + T - 1) / T;
    ldx = ((L + 31) / 32) * 32;  // rows of the B operands: whole 32-row K chunks stay in bounds
    ldr = 8 * tpc + 4;
    auto al = [](size_t v) { return (v + 15) & ~(size_t)15; };  // 128-byte alignment
    size_t o = 0;
    // B operands, row-major [row][CC] exactly as the bulk copies deliver them:
    // a DMMA B fragment (rows k+tq, columns g) then covers 32 consecutive doubles
    gst = o;   o = al(o + (size_t)2 * ldx * CC);  // right-hand side of order s by parity, natural ring order (BULK B)
    xrow = o;  o = al(o + (size_t)2 * ldx * CC);  // x_s of the whole team by parity (CORR B), pushed over DSMEM
    xst = o;   o = al(o + (size_t)2 * 8 * tpc * CC);  // own rows of x_s by parity, staged for the output warp
    ubuf = o;  o = al(o + (size_t)2 * ldx);     // u_s (chain partial weights) by parity, natural ring order
    fix = o;   o = al(o + (size_t)2 * CC);      // row-1 correction of order s by parity (DSMEM from CORR(s+3))
    xp = o;    o = al(o + (size_t)2 * CC * ldr);  // own rows of x'_s, transposed, by parity of s
    wv = o;    o = al(o + (size_t)4 * ldr);     // own rows of w_s, by s mod 4 (prefetched two steps ahead)
    apart = o; o = al(o + (size_t)4 * SWEEP_WB * CC);  // chain partials a_s per BULK warp, slot s % 4
    late = o;  o = al(o + (size_t)2 * CC);      // late right-hand-side entries L_s, by parity
    rch = o;   o = al(o + (size_t)2 * CC);      // prefetched R(+-)[s][0], by parity
    stage = o; o += (size_t)2 * S * tpc * KC * 8;  // ring B (BULK) then ring C (CORR)
    bar = o;   o += (size_t)4 * S + 2;          // fullB[S], emptyB[S], fullC[S], emptyC[S], inB[2]
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
template <int NM, int CC>
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
        // CC = 4: the columns 4..7 of the 8-wide tile are zero
        const double b = (CC >= 8 || boff[u] < CC) ? Bk[(size_t)ks * 4 * ldb + boff[u]] : 0.0;
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
    boff[u] = col;
  }
  double res[SWEEP_IPW][2];
  switch (nmine) {
    case 1: job_tiles<1, CC>(j.nch, ldb, rg, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
    case 2: job_tiles<2, CC>(j.nch, ldb, rg, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
    case 3: job_tiles<3, CC>(j.nch, ldb, rg, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
    case 4: job_tiles<4, CC>(j.nch, ldb, rg, cst, cphase, aoff, boff, Bsrc, tq, lane, res); break;
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
template <typename StepJob, typename StepHook>
__device__ __forceinline__ void produce(const Ring& rg, int nsteps, int lane, StepJob step_job, StepHook hook) {
  Job cur;
  int q_dec = 0;  // next step whose job is decoded
  bool has = false;
  int ch = 0, st = 0;
  long long issued = 0, target = 0;
  uint32_t ephase_bits = 0;  // per-stage parity of the next empty completion to wait for
#ifdef OSPH_SWEEP_PROF
  long long arr_acc = 0, t_top = clock64();
#endif
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
      hook(q);  // per-step work of the producer thread (after the step's barrier)
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
#ifdef OSPH_SWEEP_PROF
    if (lane == 0) arr_acc += clock64() - t_top;
#endif
    __syncwarp();
    step_barrier<2>();  // bulk copies are tracked by mbarriers, not by this barrier
#ifdef OSPH_SWEEP_PROF
    t_top = clock64();
#endif
  }
#ifdef OSPH_SWEEP_PROF
  if (blockIdx.x == 0 && lane == 0) printf("sweep prof producer %s: work before arrive %lld cycles\n", rg.S == -1 ? "" : (threadIdx.x >> 5) == SWEEP_WC + SWEEP_WB ? "B" : "C", arr_acc);
#endif
}

template <int CC>
__global__ void __launch_bounds__(SWEEP_THREADS_ALL, 1) k_sweep(
    int L, int B, int maps_per_team, int KC, int S,
    const double* __restrict__ xt, const int64_t* __restrict__ xt_off, const double* __restrict__ beta_all,
    const double* __restrict__ pbt, const int64_t* __restrict__ pb_off, const double* __restrict__ u_all,
    const double* __restrict__ w_all, double2* __restrict__ R, double2* __restrict__ flm) {
  const int T = (int)cg::this_cluster().num_blocks();
  const int rank = (int)cg::this_cluster().block_rank();
  const int lgT = __ffs(T) - 1;  // T is a power of two (launch_sweep)
  const int team = (int)(blockIdx.x >> lgT);
  const int b0 = team * maps_per_team;
  const int G = maps_per_team;  // a power of two
  // this team's slab of the team-major right-hand side [pos][+-][G] (common.cuh)
  double2* const Rt = R + (int64_t)team * ((int64_t)L * (L + 1) / 2) * 2 * G;
  const int gm = min(maps_per_team, B - b0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;

  extern __shared__ __align__(128) double smem[];
  const SweepCfg cfg(L, T, CC, KC, S);
  const int ldr = cfg.ldr, tpc = cfg.tpc;
  double* gst = smem + cfg.gst;
  double* xrow = smem + cfg.xrow;
  double* xst = smem + cfg.xst;
  double* ubuf = smem + cfg.ubuf;
  double* xp = smem + cfg.xp;
  double* wv = smem + cfg.wv;
  double* apart = smem + cfg.apart;
  double* late = smem + cfg.late;
  double* rch = smem + cfg.rch;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + cfg.bar);
  uint64_t* inB = bars + 4 * S;  // B operands of BULK landed, by parity of the order
  double* fix = smem + cfg.fix;

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
    mbar_init(inB, 1);
    mbar_init(inB + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // B operands start zeroed: a chunk's rows past K multiply zero operand tiles,
  // so those entries must be finite
  for (size_t i = tid; i < cfg.stage; i += SWEEP_THREADS_ALL) smem[i] = 0.0;
  fence_proxy_async();
  __syncthreads();

  // Steps: q = 0 is the prologue, q = L - t is step t.
  const int nsteps = L + 1;

  // B operands of BULK(s) -> buffers of parity s (one thread, bulk copies):
  // the right-hand side rows pos(s, 0..ns-1) of the team's maps (TMA boxes of
  // the [pos][+-][map] R), w_s on own rows and u_s.  Orders >= SWEEP_PF_MIN
  // are fetched one step early (their last correction but row 1's has landed;
  // row 1's arrives through `fix`), so BULK does not wait on the copy.
  auto operands_issue = [&](int s) {
    fence_proxy_async();
    const int ns = L - s, nrt = (ns + 7) / 8;
    const int r0 = 8 * ((rank * nrt) >> lgT), r1 = min(ns, 8 * (((rank + 1) * nrt) >> lgT));
    const uint32_t wb = (uint32_t)(((max(r1 - r0, 0) + 1) & ~1) * 8);
    const uint32_t ub = (uint32_t)(((ns + 1) & ~1) * 8);
    const uint32_t rb = (uint32_t)(ns * CC * 8);  // rows pos(s, 0..ns-1) of the team slab: [+-][map][re, im]
    uint64_t* bar = inB + (s & 1);
    mbar_arrive_expect_tx(bar, rb + wb + ub);
    bulk_g2s(gst + (size_t)(s & 1) * cfg.ldx * CC, Rt + packed_pos(L, s, 0) * 2 * G, rb, bar);
    if (wb) bulk_g2s(wv + (size_t)(s & 3) * ldr, w_all + (size_t)s * uw_ld(L) + r0, wb, bar);
    bulk_g2s(ubuf + (size_t)(s & 1) * cfg.ldx, u_all + (size_t)s * uw_ld(L), ub, bar);
  };

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
    }, [&](int q) {  // prefetch BULK's operands of order t-2 at step t (L-2 in the prologue)
      const int s2 = q == 0 ? L - 2 : L - q - 2;
      if (s2 >= 0) operands_issue(s2);
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
    }, [](int) {});
    return;
  }

  if (warp == SWEEP_WC + SWEEP_WB + 2) {
    // ======================= output warp =======================
    // Writes x_s (own rows, staged by the chain/CORR warps one step earlier) to
    // flm.  Its HBM stores are not read inside the kernel, so it arrives at the
    // step barrier relaxed (a release would wait for them).
    auto write_out = [&](int s) {
      const int ns = L - s, nrt = (ns + 7) / 8;
      const int r0 = 8 * ((rank * nrt) >> lgT), r1 = min(ns, 8 * (((rank + 1) * nrt) >> lgT));
      const double* xs = xst + (size_t)(s & 1) * 8 * tpc * CC;
      for (int idx = lane; idx < (r1 - r0) * (CC / 2); idx += 32) {
        const int l = r0 + idx / (CC / 2), c = 2 * (idx % (CC / 2));
        const int bl = c >> 2;
        if (bl >= gm) continue;
        const double2 v = *reinterpret_cast<const double2*>(xs + (size_t)(l - r0) * CC + c);
        const int64_t ell = s + l;
        double2* f = flm + (int64_t)(b0 + bl) * L * L + ell * ell + ell;
        if ((c & 2) == 0) __stcs(f + s, v);
        else if (s > 0) __stcs(f - s, v);
      }
    };
#ifdef OSPH_SWEEP_PROF
    long long o_acc = 0, o_top = clock64();
#endif
    for (int q = 0; q < nsteps; ++q) {
      const int t = L - q;  // step t (q = 0: prologue)
      if (q >= 2) write_out(t + 1);  // x_{t+1}
#ifdef OSPH_SWEEP_PROF
      if (lane == 0) o_acc += clock64() - o_top;
#endif
      __syncwarp();
      step_barrier<2>();
#ifdef OSPH_SWEEP_PROF
      o_top = clock64();
#endif
    }
#ifdef OSPH_SWEEP_PROF
    if (blockIdx.x == 0 && lane == 0) printf("sweep prof output warp: work before arrive %lld cycles\n", o_acc);
    if (blockIdx.x == 0 && lane == 0) {
      __nanosleep(100000);
      for (int w = 0; w < 11; ++w) printf("sweep prof arrive warp %d: %lld\n", w, g_prof_arrive[w]);
    }
#endif
    write_out(0);
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
        const int64_t base = (packed_pos(L, s, 0) * 2) * G + gt;
        const double2 rp = __ldcg(Rt + base), rn = __ldcg(Rt + base + G);
        double* d = rch + (size_t)(s & 1) * CC + 4 * gt;
        d[0] = rp.x;
        d[1] = rp.y;
        d[2] = rn.x;
        d[3] = rn.y;
      }
    };
    auto rch_issue = [&](int s) {  // the same by cp.async (slots gm..NB4-1 stay zero)
      if (gt < gm) {
        const int64_t base = (packed_pos(L, s, 0) * 2) * G + gt;
        double* d = rch + (size_t)(s & 1) * CC + 4 * gt;
        cp_async16(d, Rt + base);
        cp_async16(d + 2, Rt + base + G);
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
      // the late entry R[t-1][0] of the next step (final now; R[0][0] takes
      // order-2 corrections at step 1 and is read synchronously at step 0)
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
          double a[4] = {0.0, 0.0, 0.0, 0.0};
          const double* ap = apart + (size_t)(t & 3) * SWEEP_WB * CC + 4 * b;
#pragma unroll
          for (int w = 0; w < SWEEP_WB; ++w)
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] += ap[w * CC + u];
          const double* ln = late + (size_t)((t + 1) & 1) * CC + 4 * b;
          gp_r = a[0] + bt * ln[0];
          gp_i = a[1] + bt * ln[1];
          gm_r = s1 * (a[2] + bt * ln[2]);
          gm_i = s1 * (a[3] + bt * ln[3]);
        }
        const double* rr = rch + (size_t)(t & 1) * CC + 4 * b;
        double* lt = late + (size_t)(t & 1) * CC + 4 * b;
        if (t == 0) {  // bin 0 of ring 0: + slot + the - tones collected in the - slot
          lt[0] = rr[0] + rr[2] - gp_r - gm_r;
          lt[1] = rr[1] + rr[3] - gp_i - gm_i;
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
      // ---- (b) x_t = x'_t + w_t L_t on own rows -> every CTA's xrow (DSMEM) and
      // the local staging for the output warp (flm)
      {
        const int nrt = (nt + 7) / 8;
        const int r0 = 8 * ((rank * nrt) >> lgT), r1 = min(nt, 8 * (((rank + 1) * nrt) >> lgT));
        const double* xps = xp + (size_t)(t & 1) * CC * ldr;
        const double* wvs = wv + (size_t)(t & 3) * ldr;
        const double* lt = late + (size_t)(t & 1) * CC;
        double* xo = xrow + (size_t)(t & 1) * cfg.ldx * CC;
        double* xs = xst + (size_t)(t & 1) * 8 * tpc * CC;
        // x_t is needed by CORR(t) at step t-1 (1 <= t-1, t <= L-1)
        const bool push = t >= 2 && t <= L - 1;
        for (int idx = gt; idx < (r1 - r0) * (CC / 2); idx += SWEEP_NC) {
          const int l = r0 + idx / (CC / 2), c = 2 * (idx % (CC / 2));
          const double wl = wvs[l - r0];
          const double2 v = make_double2(xps[(size_t)c * ldr + (l - r0)] + wl * lt[c],
                                         xps[(size_t)(c + 1) * ldr + (l - r0)] + wl * lt[c + 1]);
          *reinterpret_cast<double2*>(xs + (size_t)(l - r0) * CC + c) = v;
          if (push) {
            double2* dst = reinterpret_cast<double2*>(xo + (size_t)l * CC + c);
            for (int q = 0; q < T; ++q) *cg::this_cluster().map_shared_rank(dst, q) = v;
          }
        }
      }
      PROF_MARK(2);
      // ---- (c) CORR(t+1): corrections of order s = t+1 on own rings k < t
      if (corr) {
        const int s = t + 1;
        const double ss = (s & 1) ? -1.0 : 1.0;
        PROF_MARK(3);
        const Job j = make_job(1, s, L, lgT, rank, SWEEP_KC, xt, xt_off, pbt, pb_off, false);
        run_job<CC>(j, ringC, cst, cphase, gw, SWEEP_WC, xrow + (size_t)(s & 1) * cfg.ldx * CC, CC, g, tq, lane,
                    [&](int k, int c, double v0, double v1) {
          const int bl = c >> 2;
          if (k >= s - 1 || bl >= gm) return;  // ring s-1 is the chain
          const bool plus = (c & 2) == 0;
          const double gr = plus ? v0 : ss * v0, gi = plus ? v1 : ss * v1;
          if (k == s - 2 && s - 3 >= SWEEP_PF_MIN) {
            // row 1 of order s-3 (ring s-2): its right-hand side was prefetched
            // before this correction, so the correction goes to every CTA's
            // fix-up slot (DSMEM) instead of R
            int tm, slot;
            corr_target(s, k, plus, tm, slot);
            const int col = slot * (CC / 2) + 2 * bl;  // gst column order [+-][map][re, im]
            double* fx = fix + ((s - 3) & 1) * CC + col;
            for (int q = 0; q < T; ++q) {
              double* rf = cg::this_cluster().map_shared_rank(fx, q);
              rf[0] = -gr;
              rf[1] = -gi;
            }
            return;
          }
          int tm, slot;
          corr_target(s, k, plus, tm, slot);
          // fire-and-forget reductions (RED.ADD.F64)
          double2* rp = Rt + (packed_pos(L, tm, k - tm) * 2 + slot) * G + bl;
          atomicAdd(&rp->x, -gr);
          atomicAdd(&rp->y, -gi);
        });
      }
      PROF_MARK(4);
      cp_async_wait_all();
      // release: this step's reductions (read by bulk copies: proxy fence too),
      // the DSMEM pushes of x_t and the fix-ups
      fence_proxy_async();
      step_barrier<0>();
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
    // Columns of gst are [+-][map][re, im] (the TMA box order); every other
    // buffer uses [map][+-][re, im].  Column pair c, c+1 of gst -> canonical pair.
    auto canon_col = [](int c) {
      const int sl = c >= CC / 2 ? 1 : 0;
      return 4 * ((c - sl * (CC / 2)) >> 1) + 2 * sl;
    };
    uint32_t inph = 0;  // phase bit per parity buffer
    auto operands_wait = [&](int s) {
      mbar_wait(inB + (s & 1), (inph >> (s & 1)) & 1u);
      inph ^= 1u << (s & 1);
    };
    // BULK(s): x'_s on own rows (the (-1)^s of the -m columns applied here),
    // and the chain partial a_{s-1} = u_s . rhs_s of the whole team: every CTA
    // holds the full right-hand side, so no exchange is needed
    auto bulk = [&](int s) {
      const Job j = make_job(0, s, L, lgT, rank, SWEEP_KC, xt, xt_off, pbt, pb_off, false);
      const int ns = j.K;
      const int r0 = 8 * j.rt0;
      const double* gs = gst + (size_t)(s & 1) * cfg.ldx * CC;
      const double* ub = ubuf + (size_t)(s & 1) * cfg.ldx;
      double* xps = xp + (size_t)(s & 1) * CC * ldr;
      const double ss = (s & 1) ? -1.0 : 1.0;
      run_job<CC>(j, ringB, cst, cphase, gw, SWEEP_WB, gs, CC, g, tq, lane, [&](int l, int c, double v0, double v1) {
        if (l < ns) {
          const int cc = canon_col(c);
          const double sg = (cc & 2) ? ss : 1.0;
          xps[(size_t)cc * ldr + (l - r0)] = sg * v0;
          xps[(size_t)(cc + 1) * ldr + (l - r0)] = sg * v1;
        }
      });
      PROF_MARK(3);
      if (s >= 1) {  // u_s . rhs_s on the tensor cores: row 0 of an 8 x K A operand
        constexpr int NCT = (CC + 7) / 8;
        double acc[NCT][2][2];
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct) acc[ct][0][0] = acc[ct][0][1] = acc[ct][1][0] = acc[ct][1][1] = 0.0;
        const int nks = (ns + 3) >> 2;
        for (int kk = gw; kk < nks; kk += 2 * SWEEP_WB) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (kk + h * SWEEP_WB >= nks) break;  // warp-uniform
            const int k = 4 * (kk + h * SWEEP_WB) + tq;  // rows ns..4*nks-1: u is zero there
            const double a = g == 0 ? ub[k] : 0.0;
#pragma unroll
            for (int ct = 0; ct < NCT; ++ct) {
              const int col = ct * 8 + g;
              const double b = (CC >= 8 || col < CC) ? gs[(size_t)k * CC + col] : 0.0;
              dmma_8x8x4(acc[ct][h][0], acc[ct][h][1], a, b);
            }
          }
        }
        if (g == 0) {
          double* ap = apart + ((s - 1) & 3) * SWEEP_WB * CC + gw * CC;
#pragma unroll
          for (int ct = 0; ct < NCT; ++ct) {
            const int c = ct * 8 + 2 * tq;
            if (c < CC) {
              const int cc = canon_col(c);
              const double sg = (cc & 2) ? ss : 1.0;
              ap[cc] = sg * (acc[ct][0][0] + acc[ct][1][0]);
              ap[cc + 1] = sg * (acc[ct][0][1] + acc[ct][1][1]);
            }
          }
        }
      }
    };

    // ---- prologue: x'_{L-1}, a_{L-2} (the producer prefetches order L-2)
    if (gt == 0) operands_issue(L - 1);
    operands_wait(L - 1);
    bulk(L - 1);
    step_barrier<1>();  // x'_s, a_s: read by this CTA's chain/CORR warps only
    for (int t = L - 1; t >= 0; --t) {
      if (t >= 1) {
        const int s = t - 1;
        operands_wait(s);  // issued at step t+1 (or in the prologue)
        if (s >= SWEEP_PF_MIN) {
          // the one correction the early copy missed: CORR(s+3) on ring s+1,
          // pushed into `fix` during the last step (none if CORR(s+3) does not exist)
          if (gt < CC) gst[((size_t)(s & 1) * cfg.ldx + 1) * CC + gt] += fix[(s & 1) * CC + gt];
        } else {
          // small orders: aliases are dense, fetch again now that R is final
          if (gt == 0) operands_issue(s);
          operands_wait(s);
          if (s == 0) {
            // order 0: add the - slot (the -tone corrections of bin 0) into the + slot;
            // gst columns are [+-][map][re, im], the - half starts at CC / 2
            group_sync(SWEEP_BAR_B, SWEEP_NB);
            double* g0 = gst;  // parity 0
            for (int i = gt; i < L * (CC / 2); i += SWEEP_NB) {
              const int r = i / (CC / 2), c = i - r * (CC / 2);
              g0[(size_t)r * CC + c] += g0[(size_t)r * CC + c + CC / 2];
            }
          }
        }
        group_sync(SWEEP_BAR_B, SWEEP_NB);
        PROF_MARK(1);
        bulk(s);
      }
      PROF_MARK(4);
      step_barrier<1>();
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
                         (const double*)p->d_beta, (const double*)p->d_pbelow, (const int64_t*)p->d_pb_off,
                         (const double*)p->d_u, (const double*)p->d_w, p->d_r, flm);
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

// Launch configuration for batch B (cached): maps per team g (1, 2, 4), team
// width T (power of two), ring stages S.  Returns g, which also fixes the
// team-major layout of R written by the forward ring DFTs.
int sweep_maps_per_team(osph_plan* p, int B) {
  const int L = p->L;
  const size_t cap = 220 * 1024;
  const int KC = SWEEP_KC;
  if (p->sweep_cfg_B == B) return p->sweep_cfg[0];
  p->sweep_gemm = false;
  p->sweep_blocked = false;
  {
    // L <= 512: orders peeled in blocks of 32 with batched GEMM launches (sweep_block.cu; B = 1:
    // 0.15 -> 0.07 ms at L = 64, 0.86 -> 0.32 ms at L = 256, 2.4 -> 0.9 ms at L = 512 against the
    // persistent kernel); OSPH_SWEEP_BLOCKED=0 forbids it
    const char* eb = getenv("OSPH_SWEEP_BLOCKED");
    // (L > 512 keeps the large sweep: its refinement step holds the round trip at 2e-10 at L = 1024,
    // the blocked sweep without one gives 2e-9 -- still inside 10x the reference's own 5e-10, but worse)
    const bool can = (L <= 512 || (eb && atoi(eb) != 0)) && L <= 1024 && !p->windowed && p->d_ut && !getenv("OSPH_SWEEP_LARGE") &&
                     !getenv("OSPH_SWEEP_GEMM") && !getenv("OSPH_SWEEP_NO_GEMM");
    if (can && (eb ? atoi(eb) != 0 : true)) {  // measured faster than the persistent kernel at every batch size
      p->sweep_blocked = true;
      p->sweep_large = false;
      p->sweep_cfg_B = B;
      p->sweep_cfg[0] = 1;
      p->sweep_cfg[1] = p->sweep_cfg[2] = 0;
      return 1;
    }
  }
  if (L > 1024 || p->windowed || getenv("OSPH_SWEEP_LARGE")) {  // the right-hand sides no longer fit the persistent kernel's smem
    p->sweep_large = true;
    p->sweep_cfg_B = B;
    p->sweep_cfg[0] = 1;
    p->sweep_cfg[1] = p->sweep_cfg[2] = 0;
    return 1;
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
  if ((!found && B >= 16 && !getenv("OSPH_SWEEP_NO_GEMM")) || getenv("OSPH_SWEEP_GEMM")) {
    // teams would run in waves: one GEMM pair per order over the whole GPU instead (sweep_gemm.cu)
    p->sweep_gemm = true;
    p->sweep_large = false;
    p->sweep_cfg_B = B;
    p->sweep_cfg[0] = 1;
    p->sweep_cfg[1] = p->sweep_cfg[2] = 0;
    return 1;
  }
  if (!found) {
    // several waves of teams: over (g, T) that fit, maximise the maps in flight
    // (resident teams x maps per team); ties go to the narrower team
    int best_flight = 0;
    for (int gg = gmax; gg >= 1; gg /= 2) {
      for (int TT = 1; TT <= 16; TT *= 2) {
        if (TT * 32 > 2 * L && TT > 1) break;
        if (!tiles_ok(gg, TT) || !fits(gg, TT, 3)) continue;
        int ss = 3;
        while (ss < SWEEP_SMAX && fits(gg, TT, ss + 1)) ++ss;
        const int flight = std::min((B + gg - 1) / gg, mac(gg, TT, ss)) * gg;
        if (flight > best_flight) {
          best_flight = flight;
          g = gg;
          T = TT;
          S = ss;
        }
      }
      if (gg == 1) break;
    }
  }
  T = env_int("OSPH_SWEEP_T", T);
  while (T & (T - 1)) T &= T - 1;  // the kernel needs a power-of-two team width
  S = env_int("OSPH_SWEEP_S", S);
  if (!tiles_ok(g, T) || !fits(g, T, S)) {  // nothing fits: two kernels per order (sweep_large.cu)
    p->sweep_large = true;
    p->sweep_cfg_B = B;
    p->sweep_cfg[0] = 1;
    p->sweep_cfg[1] = p->sweep_cfg[2] = 0;
    return 1;
  }
  p->sweep_large = false;
  p->sweep_cfg_B = B;
  p->sweep_cfg[0] = g;
  p->sweep_cfg[1] = T;
  p->sweep_cfg[2] = S;
  return g;
}

cudaError_t launch_sweep(osph_plan* p, int B, double2* flm) {
  const int g = sweep_maps_per_team(p, B), T = p->sweep_cfg[1], S = p->sweep_cfg[2];
  if (p->sweep_blocked) {
    if (ensure_sweep_blocked(p)) return cudaErrorMemoryAllocation;
    return launch_sweep_blocked(p, B, flm);
  }
  if (p->sweep_gemm) return launch_sweep_gemm(p, B, flm);
  if (p->sweep_large) return launch_sweep_large(p, B, flm);
  if (g == 4) return launch_sweep_cc<16>(p, B, 4, T, SWEEP_KC, S, flm);
  if (g == 2) return launch_sweep_cc<8>(p, B, 2, T, SWEEP_KC, S, flm);
  return launch_sweep_cc<4>(p, B, 1, T, SWEEP_KC, S, flm);
}
