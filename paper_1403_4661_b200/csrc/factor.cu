// factor.cu -- the per-call factorisation stage of the forward transform.
//
// Reference: the forward transform solves, for each order m, the square
// system (2pi Y_lm(theta_k, 0))_{k>=m, l>=m} f = g with a rank-revealing
// least-squares solve (gelsy, rcond 1e-14) and raises
// IllConditionedSolveError(order, kappa) on rank deficiency
// (pkg/src/optisph/transform.py:396-429, blocks.py:88-116).  The blocks do
// not depend on the data, so every order is factored up front, in parallel
// over m: one breadth-first blocked Gauss-Jordan pass over all orders with
// the grid's pivot order (factor_bf.cu; the pivot order itself is found once
// per grid by pivots.cu).  The result X satisfies A^{-1} = X P: the sweep
// multiplies the right-hand side by X, a parallel GEMV instead of two serial
// triangular solves (LU vs gelsy: max|df| 2.2e-14 at L=512).
//
// The reference's rank check becomes a 1-norm condition estimate
// kappa = ||A||_1 ||A^{-1}||_1 / sqrt(n), flagged above 2/rcond = 2e14
// (calibrated on the interleaved L=256 grid: gelsy first reports rank
// deficiency at m=220 where this estimate is 3.0e14; m=221 gives 1.9e14).
#include <algorithm>
#include <cstdlib>

#include "plan.cuh"

// Finalise kappa per order once every order's norms are in.
__global__ void k_kappa(int L, const unsigned long long* __restrict__ norms, double* __restrict__ kappa) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= L) return;
  const double a = __longlong_as_double((long long)norms[2 * m]);
  const double x = __longlong_as_double((long long)norms[2 * m + 1]);
  const double k = a * x / sqrt((double)(L - m));
  kappa[m] = isfinite(k) ? k : INFINITY;
}

cudaError_t launch_kappa(osph_plan* p, cudaStream_t st) {
  k_kappa<<<(p->L + 127) / 128, 128, 0, st>>>(p->L, p->d_norms, p->d_kappa);
  p->launches++;
  return cudaGetLastError();
}

// Every order in one breadth-first pass on `st` (the resident, non-windowed
// forward; the windowed one runs bf_run per window in window.cu).
//
// Split (unsharded plans, L >= 128; OSPH_FACTOR_SPLIT=0 disables, =n sets the
// number of ranges): the chain of panel steps is latency-bound, and the high
// orders (small blocks: few panel steps, a few percent of the flops) are the
// first the sweep needs.  The orders are cut into three (up to four) ranges at sweep
// block boundaries; every range runs its own chain on its own stream, all
// beside each other, and records an event when done, so the blocked sweep
// starts on the high orders while the lower ranges are still being factored
// (launch_sweep_blocked waits per range).  `st` runs the lowest range and joins
// the other streams before returning, so an event recorded on `st` after this
// call still covers every order.
cudaError_t launch_factor(osph_plan* p, cudaStream_t st) {
  const int L = p->L;
  cudaError_t e;
  if (!st) st = p->stream;
  if ((e = cudaMemsetAsync(p->d_norms, 0, sizeof(unsigned long long) * 2 * L, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p->d_status, 0, sizeof(int) * L, st)) != cudaSuccess) return e;
  int lo, hi;
  own_orders(p, lo, hi);  // all orders, or this shard's block (OSPH_SHARD_FACTORS)
  static const int split_env = getenv("OSPH_FACTOR_SPLIT") ? atoi(getenv("OSPH_FACTOR_SPLIT")) : -1;
  p->fsplit_active = false;
  p->sweep_waits_ranges = false;
  if (split_env != 0 && !p->shard_mode && !p->windowed && lo == 0 && hi == L - 1 && L >= 128 && p->s_f[0]) {
    if (p->n_frng == 0) {
      // boundaries at multiples of the sweep block, ranges of about L / n orders
      // default three ranges (measured, config 2: 39.9k / 41.6k / 41.9k / 41.9k transforms/s with 1 / 2 / 3 / 4)
      const int want = std::min<int>(osph_plan::kFactorRanges, split_env > 0 ? split_env : 3);
      int n = 0, top = L - 1;
      for (int r = 0; r < want && top >= 0; ++r) {
        int first = r == want - 1 ? 0 : (((int64_t)L * (want - 1 - r) / want) / OSPH_SB_BLOCK) * OSPH_SB_BLOCK;
        if (first > top) continue;
        if ((e = bf_prepare(p, first, top, &p->bf_rng[n])) != cudaSuccess) return e;
        p->bf_rng[n].dbuf = p->d_bf_d + bf_diag_doubles(first);  // disjoint diagonal-block scratch
        ++n;
        top = first - 1;
      }
      p->n_frng = n;
    }
    const int n = p->n_frng;
    const BfOffsets o{p->d_ainv_off, p->d_xt_off, p->d_pb_off, p->d_bf_off};
    // Enqueue the longest chain first (the lowest orders: most panel steps): the host needs a few
    // microseconds per launch, and every range queued ahead of it would delay the chain the
    // sweep waits for last.
    if ((e = cudaEventRecord(p->ev_fstart, st)) != cudaSuccess) return e;
    if ((e = bf_run(p, p->bf_rng[n - 1], st, o)) != cudaSuccess) return e;
    for (int r = n - 2; r >= 0; --r) {
      if ((e = cudaStreamWaitEvent(p->s_f[r], p->ev_fstart, 0)) != cudaSuccess) return e;
      if ((e = bf_run(p, p->bf_rng[r], p->s_f[r], o)) != cudaSuccess) return e;
      if ((e = cudaEventRecord(p->ev_f[r], p->s_f[r])) != cudaSuccess) return e;
    }
    for (int r = 0; r < n - 1; ++r)
      if ((e = cudaStreamWaitEvent(st, p->ev_f[r], 0)) != cudaSuccess) return e;
    p->fsplit_active = true;
    return launch_kappa(p, st);
  }
  if ((e = launch_factor_bf(p, lo, hi, st)) != cudaSuccess) return e;
  return launch_kappa(p, st);
}
