/*
 * osph.h -- C ABI of libosph.so, the B200 (sm_100a) forward/inverse spherical
 * harmonic transform on the optimal-dimensionality L^2-sample grid.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (optisph, pure Python) has no C ABI of its own; its callers bind the Python
 * functions re-exported from optisph/__init__.py:39-48.  Each entry point
 * below replaces one of them:
 *
 *   osph_plan_create   <- the per-band-limit precomputation the reference
 *                         caches implicitly: _packed_tables / _ring_roots_flat
 *                         (pkg/src/optisph/transform.py:268-301) plus the grid
 *                         co-latitudes ColatitudeGrid.thetas (sampling.py:46-79)
 *   osph_inverse       <- inverse_sht(coeffs, grid)      (transform.py:347-357)
 *   osph_forward       <- forward_sht(samples, grid, method, check, stats)
 *                                                        (transform.py:360-393)
 *   osph_stats         <- TransformStats                 (transform.py:106-112)
 *   OSPH_ERR_*         <- BandLimitError / IllConditionedSolveError(order, kappa)
 *                         (errors.py:8-36; raised at transform.py:134-136 and
 *                         blocks.py:113-115)
 *
 * Data layouts are the reference's flat layouts, so host<->device copies are
 * plain memcpys:
 *   coefficients  complex128 [B][L*L], index l*l + l + m   (transform.py:41-43)
 *   samples       complex128 [B][L*L], ring k at [k*k, (k+1)*(k+1)),
 *                 sample j of ring k at phi_j = 2*pi*j/(2k+1)  (transform.py:87-96)
 * Complex values are interleaved (re, im) doubles, identical to numpy complex128.
 *
 * Conventions: a plan is bound to one CUDA device and is used by one host
 * thread at a time; concurrent plans are allowed.  Inputs are never modified.
 * All calls are host-blocking (results valid on return) unless OSPH_ASYNC is
 * set together with OSPH_DEVICE, in which case work is enqueued on the plan's
 * stream and the caller synchronises.  Every entry point returns an OSPH_*
 * code; osph_last_error() gives a thread-local message for the last failure.
 */
#ifndef OSPH_H
#define OSPH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OSPH_ABI_VERSION 3

/* return codes */
#define OSPH_OK 0
#define OSPH_ERR_ARG 1        /* band-limit mismatch / bad argument (BandLimitError, ValueError) */
#define OSPH_ERR_ILLCOND 2    /* per-order block numerically singular (IllConditionedSolveError) */
#define OSPH_ERR_CUDA 3       /* CUDA runtime failure (no device, launch error, OOM) */
#define OSPH_ERR_NCCL 4       /* inter-GPU exchange failed (peer copy / collective of a multi-GPU plan) */
#define OSPH_ERR_ORDER 5      /* order / spin outside the band limit (OrderRangeError) */

/* pointer kinds / flags for osph_inverse / osph_forward */
#define OSPH_HOST 0   /* host pointers: the library copies in and out (pinned memory is fastest) */
#define OSPH_DEVICE 1 /* device pointers on the plan's device */
#define OSPH_ASYNC 2  /* with OSPH_DEVICE: enqueue on the plan stream and return immediately */
#define OSPH_REAL 4   /* real-valued maps: flm conjugate-symmetric (f_{l,-m} = (-1)^m conj f_lm) /
                         samples real (imaginary parts ignored); layouts unchanged (complex128),
                         output samples have zero imaginary parts.  Pairs of maps run as one
                         complex transform (half the work); results equal the complex path's
                         to rounding. */

typedef struct osph_plan osph_plan;

/* Mirrors optisph.transform.TransformStats (transform.py:106-112) plus the
 * failure payload of IllConditionedSolveError (errors.py:28-36). */
typedef struct osph_stats {
  double solve_seconds;   /* device time of the per-order solve stage (factor + sweep) */
  int32_t orders;         /* number of orders processed (= L) */
  int32_t failed_order;   /* highest order whose block failed the check, -1 if none */
  double failed_kappa;    /* infinity-norm condition estimate of that block */
  double factor_seconds;  /* device time of the batched per-order factorisation */
  double sweep_seconds;   /* device time of the order-peeling sweep */
  double total_seconds;   /* device time of the whole call */
} osph_stats;

/* Create a plan for band limit L on ndev devices devs[0..ndev-1].
 * thetas[L] are the ring co-latitudes (ColatitudeGrid.thetas, ring k = ring
 * with 2k+1 samples).  max_batch bounds B in later calls (workspace is sized
 * for it).  ndev = 1: one device.  ndev > 1: one host thread drives every
 * device (devices may repeat, e.g. for tests); osph_inverse / osph_forward
 * then shard the work:
 *   B >= ndev   maps split over the devices; the forward's per-order
 *               factorisation is split by order blocks and the factors are
 *               copied peer to peer to every device (no redundant factoring);
 *   B <  ndev   one map chain: the inverse is split by ring ranges, the
 *               forward by load-balanced blocks of orders m, each device
 *               factoring its own block while the sweep passes the corrected
 *               ring spectra and the completed coefficients from block to
 *               block (peer copies over NVLink).
 * Host pointers only for ndev > 1 (the plan owns every device's buffers). */
int osph_plan_create(int L, const double* thetas, int max_batch, int ndev, const int* devs, osph_plan** out);
int osph_plan_destroy(osph_plan* plan);

/* Use `stream` (a cudaStream_t) for all work of this plan; NULL = plan-owned
 * stream (pass cudaStreamLegacy, i.e. (void*)1, for the legacy default stream). */
int osph_plan_set_stream(osph_plan* plan, void* stream);

/* Band limit / batch capacity of a plan. */
int osph_plan_info(const osph_plan* plan, int* L, int* max_batch);

/* inverse_sht for B maps: flm [B][L*L] complex128 -> samples [B][L*L] complex128. */
int osph_inverse(osph_plan* plan, int B, const void* flm, void* samples, int ptr_kind);

/* forward_sht for B maps: samples [B][L*L] -> flm [B][L*L].
 * check != 0 refuses numerically singular per-order blocks (OSPH_ERR_ILLCOND,
 * stats->failed_order / failed_kappa filled).  stats may be NULL. */
int osph_forward(osph_plan* plan, int B, const void* samples, void* flm, int ptr_kind, int check,
                 osph_stats* stats);

/* ring_analysis(ring_values, m) (transform.py:115-131) for one host ring of odd
 * length n: out[0..1] = delta * sum_j v_j e^{-i m phi_j} (re, im),
 * out[2..3] = delta * sum_j v_j e^{+i m phi_j}, delta = 2 pi / n.  Refuses
 * |m| > (n-1)/2 (AliasingError) and even n with OSPH_ERR_ARG. */
int osph_ring_analysis(const double* ring, int n, int m, double* out, int device);

/* legendre_table(m, grid.thetas, L) (legendre.py:110-143) on the device for
 * all L plan rings: out[(l - m) * ld + k] = Y_lm(theta_k, 0) for l = m..L-1,
 * k < L (degree-major; ld >= L).  Values below 2^-500 are returned as 0.
 * ptr_kind must include OSPH_DEVICE (OSPH_ASYNC: enqueue on the plan stream).
 * Used by the grid optimiser (optimize_order, sampling.py:217-278). */
int osph_legendre_block(osph_plan* plan, int m, double* out, int64_t ld, int ptr_kind);

/* Device time of the stages of the last inverse and the last forward call, in
 * seconds: seconds[0..2] = inverse {pack, Legendre synthesis, ring inverse DFTs},
 * seconds[3..5] = forward {ring forward DFTs, per-order factorisation, sweep}
 * (0 for a direction not yet run).  Blocks until that work has finished. */
int osph_last_stage_times(const osph_plan* plan, double* seconds /* [6] */);

/* Number of kernel launches enqueued by the last osph_inverse/osph_forward call. */
int osph_last_launch_count(const osph_plan* plan);

/* Which order-peeling sweep the last osph_forward ran (the chain of
 * transform.py:441-463), or -1 before the first forward:
 *   OSPH_SWEEP_PERSISTENT  one persistent cluster kernel (sweep.cu; L <= 1024, teams resident)
 *   OSPH_SWEEP_GEMM        two whole-GPU DMMA GEMM launches per order (sweep_gemm.cu; large batches)
 *   OSPH_SWEEP_LARGE       two launches per order + refinement (sweep_large.cu; L > 1024)
 *   OSPH_SWEEP_WINDOWED    factor + large sweep window by window (window.cu; factors exceed HBM)
 *   OSPH_SWEEP_BLOCKED     orders peeled in blocks of 32: in-block aliasing resolved by a scalar
 *                          recurrence, three batched DMMA GEMM launches per block (sweep_block.cu; batches) */
#define OSPH_SWEEP_PERSISTENT 0
#define OSPH_SWEEP_GEMM 1
#define OSPH_SWEEP_LARGE 2
#define OSPH_SWEEP_WINDOWED 3
#define OSPH_SWEEP_BLOCKED 4
int osph_last_sweep_kind(const osph_plan* plan);

/* The grid's pivot order: perm[L(L+1)/2] (may be NULL), packed by order as
 * perm[m*L - m(m-1)/2 + i] = ring offset (k - m) of pivot position i of order
 * m's block -- the row order LU with partial pivoting (LAPACK getrf) picks for
 * 2pi Y_lm(theta_k), k, l >= m (the blocks gelsy solves in blocks.py:88-116).
 * Found on the first call that needs it (hand-written kernels, pivots.cu) and
 * cached per grid; *seconds (may be NULL) = wall time this plan spent finding
 * it (0 when the grid's order was already cached). */
int osph_plan_pivots(osph_plan* plan, int32_t* perm, double* seconds);

/* Thread-local description of the last error (empty string if none). */
const char* osph_last_error(void);

/* ---- one process per GPU (torch.distributed / MPI drive the exchange) ----
 * A single-device plan becomes rank `rank` of `nranks` (before its first
 * forward):
 *   OSPH_SHARD_CHAIN    one map (or a few) across GPUs: this plan factors and
 *                       sweeps only its block of orders [m_lo, m_hi] (blocks
 *                       descend in m with the rank: rank 0 owns the highest
 *                       orders, cost-balanced by sum (L-m)^3) and its inverse
 *                       synthesises only its rings [k_lo, k_hi).  Forward:
 *                       RINGS|FACTOR, receive the spectra + coefficients from
 *                       rank-1, SWEEP, send them to rank+1; the last rank
 *                       holds every coefficient (transform.py:441-463 run as
 *                       nranks consecutive blocks).
 *   OSPH_SHARD_FACTORS  batches: FACTOR factors only [m_lo, m_hi]; the
 *                       factor buffers are all-gathered (osph_shard_buffer);
 *                       then RINGS|SWEEP transforms this rank's own maps.
 * Returns OSPH_ERR_ARG if the plan already ran a forward. */
#define OSPH_SHARD_CHAIN 1
#define OSPH_SHARD_FACTORS 2
int osph_plan_shard(osph_plan* plan, int rank, int nranks, int mode);

/* The block of `rank` of `nranks` (no plan needed): orders [m_lo, m_hi] and
 * rings [k_lo, k_hi) (rings only split in chain mode). */
int osph_shard_range(int L, int rank, int nranks, int mode, int* m_lo, int* m_hi, int* k_lo, int* k_hi);

/* Forward transform in stages (device pointers; OSPH_ASYNC allowed):
 * RINGS = ring DFTs of every ring of `samples` into the plan's spectra,
 * FACTOR = factorisation of the plan's orders, SWEEP = the order-peeling
 * sweep over the plan's orders (chain shards: their block, reading and
 * updating the spectra and writing their orders of flm; otherwise every
 * order).  osph_forward == RINGS|FACTOR|SWEEP on an unsharded plan.  check
 * applies to the plan's own orders (SWEEP stage). */
#define OSPH_STAGE_RINGS 1
#define OSPH_STAGE_FACTOR 2
#define OSPH_STAGE_SWEEP 4
int osph_forward_stage(osph_plan* plan, int stages, int B, const void* samples, void* flm, int ptr_kind, int check,
                       osph_stats* stats);

/* Device address and byte size of a plan buffer the shards exchange:
 * OSPH_BUF_SPECTRA: the ring spectra of B maps (chain hand-off; m_lo/m_hi ignored);
 * the others: the factor data of orders [m_lo, m_hi] (one contiguous run each). */
#define OSPH_BUF_SPECTRA 0
#define OSPH_BUF_XT 1     /* X_m = A_m^-1, 8-row tiles */
#define OSPH_BUF_PB 2     /* 2pi Y_lm(theta_k), rings k < m, tiles */
#define OSPH_BUF_AT 3     /* A_m (refinement, L > 512; 0 bytes otherwise) */
#define OSPH_BUF_U 4      /* chain weights u_m */
#define OSPH_BUF_W 5      /* late-ring columns w_m */
#define OSPH_BUF_BETA 6   /* beta_m */
#define OSPH_BUF_JSTAR 7  /* j*_m */
#define OSPH_BUF_NORMS 8  /* ||A_m||_1, ||X_m||_1 (condition estimate) */
#define OSPH_BUF_STATUS 9 /* zero-pivot flags */
#define OSPH_BUF_UT 10    /* coupling rows U_m of the blocked sweep, tiles */
#define OSPH_BUF_COUNT 11
int osph_shard_buffer(osph_plan* plan, int which, int B, int m_lo, int m_hi, void** ptr, int64_t* bytes);

/* ---- spin-weighted transforms ----
 * spin_inverse_sht / spin_forward_sht (transform.py:474-533) on a
 * single-device, unsharded plan; layouts as osph_inverse / osph_forward.
 * spin = 0 IS the scalar path (osph_inverse / osph_forward, bit for bit);
 * |spin| >= L -> OSPH_ERR_ORDER.  Coefficients with degree l < |spin| are
 * ignored by the inverse and come back as exact zeros from the forward.  The
 * forward solves, per order m = L-1..0, the +m and -m blocks
 * 2pi sY_l(+-m)(theta_k), k >= m, l >= max(m, |spin|) separately (tall
 * least-squares blocks for m < |spin|); their solution operators are built on
 * the first forward of each spin (the plan keeps the two most recent spins) and
 * stats->factor_seconds reports that build (0 once cached).  check != 0
 * refuses a block whose condition estimate ||A||_1 ||X||_1 exceeds 2e14
 * (failed_order = the signed order).  ptr_kind: OSPH_HOST or OSPH_DEVICE
 * (| OSPH_ASYNC); OSPH_REAL is not accepted. */
int osph_spin_inverse(osph_plan* plan, int spin, int B, const void* flm, void* samples, int ptr_kind);
int osph_spin_forward(osph_plan* plan, int spin, int B, const void* samples, void* flm, int ptr_kind, int check,
                      osph_stats* stats);

/* spin_table(spin, m, grid.thetas, L) (legendre.py:276-306) on the device for
 * all L plan rings: out[(l - lo) * ld + k] = sY_lm(theta_k, 0), l = lo..L-1,
 * lo = max(|m|, |spin|) (m signed; ld >= L; values below 2^-500 returned as 0).
 * lo >= L -> OSPH_ERR_ORDER.  ptr_kind must include OSPH_DEVICE. */
int osph_spin_block(osph_plan* plan, int spin, int m, double* out, int64_t ld, int ptr_kind);

/* Host-only: the constants the spin recurrence of (spin, m) starts from at
 * degree j = max(|m|, |spin|) (legendre.py:233-262): the seed is
 * scale * 2^offset * sin(theta/2)^exp_sin * cos(theta/2)^exp_cos, scale
 * rounded from the exact rational as the reference's Fraction arithmetic.
 * Any output pointer may be NULL.  No device needed. */
int osph_spin_seed(int spin, int m, int* j, double* scale, int* offset, int* exp_sin, int* exp_cos);

/* ABI version (OSPH_ABI_VERSION) -- lets bindings refuse a mismatched library. */
int osph_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* OSPH_H */
