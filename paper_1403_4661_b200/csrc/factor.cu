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
// Split (unsharded plans, L >= 128; OSPH_FACTOR_SPLIT=0 disables): the chain of
// panel steps is latency-bound, and the orders >= L/2 (blocks of at most L/2
// rows, ~6% of the flops, half of the panel steps) are the first the sweep
// needs.  They run as their own range on a second stream beside the low
// orders; `ev_fa` marks them done, so the blocked sweep starts on the high
// orders while the low ones are still being factored.  `st` joins the second
// stream before returning, so an event recorded on `st` after this call still
// covers every order.
cudaError_t launch_factor(osph_plan* p, cudaStream_t st) {
  const int L = p->L;
  cudaError_t e;
  if (!st) st = p->stream;
  if ((e = cudaMemsetAsync(p->d_norms, 0, sizeof(unsigned long long) * 2 * L, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p->d_status, 0, sizeof(int) * L, st)) != cudaSuccess) return e;
  int lo, hi;
  own_orders(p, lo, hi);  // all orders, or this shard's block (OSPH_SHARD_FACTORS)
  static const bool split_off = getenv("OSPH_FACTOR_SPLIT") && atoi(getenv("OSPH_FACTOR_SPLIT")) == 0;
  p->fsplit_active = false;
  p->sweep_late_ev = nullptr;
  if (!split_off && !p->shard_mode && !p->windowed && lo == 0 && hi == L - 1 && L >= 128 && p->s_fa) {
    const int split = ((L / 2) / OSPH_SB_BLOCK) * OSPH_SB_BLOCK;  // a block boundary of the blocked sweep
    if (p->fsplit_m != split) {
      if ((e = bf_prepare(p, split, L - 1, &p->bf_hi)) != cudaSuccess) return e;
      if ((e = bf_prepare(p, 0, split - 1, &p->bf_lo)) != cudaSuccess) return e;
      p->bf_hi.dbuf = p->d_bf_d + bf_diag_doubles(split);  // disjoint diagonal-block scratch
      p->bf_lo.dbuf = p->d_bf_d;
      p->fsplit_m = split;
    }
    const BfOffsets o{p->d_ainv_off, p->d_xt_off, p->d_pb_off, p->d_bf_off};
    if ((e = cudaEventRecord(p->ev_fstart, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(p->s_fa, p->ev_fstart, 0)) != cudaSuccess) return e;
    if ((e = bf_run(p, p->bf_hi, p->s_fa, o)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(p->ev_fa, p->s_fa)) != cudaSuccess) return e;
    if ((e = bf_run(p, p->bf_lo, st, o)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st, p->ev_fa, 0)) != cudaSuccess) return e;
    p->fsplit_active = true;
    return launch_kappa(p, st);
  }
  if ((e = launch_factor_bf(p, lo, hi, st)) != cudaSuccess) return e;
  return launch_kappa(p, st);
}
