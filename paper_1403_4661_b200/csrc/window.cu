// window.cu -- storage of the per-order factors, and the windowed forward for
// band limits whose factors do not fit in HBM at once.
//
// Per order m (n = L - m) the forward needs the explicit inverse X_m (n^2
// doubles, plus its chunk-major tiled copy for the sweep) and the below-block
// Pb_m (m n doubles): at L = 4096 that is ~2 x 183 + 92 GB, beyond one
// B200's 180 GB.  The blocks are data independent, but the sweep consumes
// them strictly in descending m, so the orders are cut into
// windows [m_lo, m_hi] of bounded storage: factor the window (breadth-first,
// factor_bf.cu), sweep its orders (sweep_large.cu), reuse the buffers for the
// next window.  Results are identical to the non-windowed path (same kernels,
// same per-order arithmetic); only the placement of the factors changes.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/osph.h"
#include "plan.cuh"

void osph_set_error(const std::string& msg);

static int64_t order_doubles(int L, int m, bool refine) {
  const int n = L - m;
  return (int64_t)n * n + tile_size(n, n) * (refine ? 2 : 1) + tile_size(m, n) + 4 * bf_panel_doubles(n);
}

#define W_TRY(expr)                                                                  \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      osph_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));            \
      return OSPH_ERR_CUDA;                                                          \
    }                                                                                \
  } while (0)

// Offsets of the factor buffers for orders [m_first, m_last]; everything else 0.
static void range_offsets(int L, int m_first, int m_last, std::vector<int64_t>& ainv, std::vector<int64_t>& xt,
                          std::vector<int64_t>& pb, std::vector<int64_t>& bf, int64_t tot[4]) {
  ainv.assign(L + 1, 0);
  xt.assign(L + 1, 0);
  pb.assign(L + 1, 0);
  bf.assign(L + 1, 0);
  int64_t a = 0, x = 0, q = 0, b = 0;
  for (int m = m_first; m <= m_last; ++m) {
    const int n = L - m;
    ainv[m] = a;
    xt[m] = x;
    pb[m] = q;
    bf[m] = b;
    a += (int64_t)n * n;
    x += tile_size(n, n);
    q += tile_size(m, n);
    b += bf_panel_doubles(n);
  }
  tot[0] = a;
  tot[1] = x;
  tot[2] = q;
  tot[3] = b;
}

template <typename T>
static cudaError_t dalloc_w(T** ptr, size_t count) {
  return cudaMalloc((void**)ptr, sizeof(T) * std::max<size_t>(count, 1));
}

// Allocate the factor storage; decide whether the forward runs windowed.
int alloc_factor_storage(osph_plan* p) {
  const int L = p->L;
  cudaStream_t st = p->stream;
  {
    // refinement steps per order in the large-L sweep: one for L > 512 (where that
    // sweep can run; measured L=1024: 2.5e-9 -> 3.2e-10, a second step adds nothing)
    const char* r = getenv("OSPH_REFINE");
    p->refine = r ? std::max(0, atoi(r)) : (L > 512 ? 1 : 0);
  }
  const bool rf = p->refine > 0;
  int64_t full = 0;
  for (int m = 0; m < L; ++m) full += order_doubles(L, m, rf);
  size_t free_b = 0, total_b = 0;
  W_TRY(cudaMemGetInfo(&free_b, &total_b));
  const char* env_budget = getenv("OSPH_WINDOW_GB");  // testing: force a window budget
  const double budget_b = env_budget ? atof(env_budget) * 1e9 : 0.55 * (double)free_b;
  p->windowed = (double)full * 8.0 > budget_b || env_budget != nullptr;
  int own_lo, own_hi;
  own_orders(p, own_lo, own_hi);
  if (p->shard_mode == OSPH_SHARD_CHAIN) {
    // a chain shard stores (in windows) only the orders it owns
    p->windowed = true;
  } else if (p->shard_mode == OSPH_SHARD_FACTORS && p->windowed) {
    osph_set_error("factor-sharded batches need every order's factors resident (L too large for this GPU)");
    return OSPH_ERR_ARG;
  }
  std::vector<int64_t> ao, xo, po, bo;
  int64_t tot[4];
  if (!p->windowed) {
    // every order resident: offsets over all orders
    range_offsets(L, 0, L - 1, ao, xo, po, bo, tot);
    p->h_ainv_off = ao;
    p->h_xt_off = xo;
    p->h_pb_off = po;
    p->h_ainv_off[L] = tot[0];
    p->h_xt_off[L] = tot[1];
    p->h_pb_off[L] = tot[2];
    W_TRY(cudaMalloc(&p->d_ainv_off, sizeof(int64_t) * (L + 1)));
    W_TRY(cudaMalloc(&p->d_xt_off, sizeof(int64_t) * (L + 1)));
    W_TRY(cudaMalloc(&p->d_pb_off, sizeof(int64_t) * (L + 1)));
    W_TRY(cudaMalloc(&p->d_bf_off, sizeof(int64_t) * (L + 1)));
    W_TRY(cudaMemcpy(p->d_ainv_off, p->h_ainv_off.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice));
    W_TRY(cudaMemcpy(p->d_xt_off, p->h_xt_off.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice));
    W_TRY(cudaMemcpy(p->d_pb_off, p->h_pb_off.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice));
    W_TRY(cudaMemcpy(p->d_bf_off, bo.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice));
    W_TRY(dalloc_w(&p->d_ainv, (size_t)tot[0]));
    W_TRY(dalloc_w(&p->d_xt, (size_t)tot[1]));
    if (rf) W_TRY(dalloc_w(&p->d_at, (size_t)tot[1]));
    W_TRY(dalloc_w(&p->d_pbelow, (size_t)tot[2]));
    W_TRY(dalloc_w(&p->d_bf_e, (size_t)tot[3]));
    W_TRY(dalloc_w(&p->d_bf_e2, (size_t)tot[3]));
    W_TRY(dalloc_w(&p->d_bf_r, (size_t)(2 * tot[3])));  // two R buffers (alternating steps), zeroed once
    W_TRY(cudaMemsetAsync(p->d_bf_r, 0, sizeof(double) * (size_t)(2 * tot[3]), st));
    p->bf_r_half = tot[3];
    W_TRY(dalloc_w(&p->d_bf_d, (size_t)bf_diag_doubles(L)));
    // padding of the tiled operands stays zero forever (the kernels write only real entries)
    W_TRY(cudaMemsetAsync(p->d_pbelow, 0, sizeof(double) * (size_t)tot[2], st));
    W_TRY(cudaMemsetAsync(p->d_xt, 0, sizeof(double) * (size_t)tot[1], st));
    // coupling rows of the blocked sweep (rows past the rings below s and padding stay zero)
    if (L > 1024) return OSPH_OK;  // the blocked sweep serves L <= 1024
    p->h_ut_off.assign(L + 1, 0);
    for (int m = 0; m < L; ++m) p->h_ut_off[m + 1] = p->h_ut_off[m] + tile_size(sb_rows(m), L - m);
    W_TRY(cudaMalloc(&p->d_ut_off, sizeof(int64_t) * (L + 1)));
    W_TRY(cudaMemcpy(p->d_ut_off, p->h_ut_off.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice));
    W_TRY(dalloc_w(&p->d_ut, (size_t)p->h_ut_off[L]));
    W_TRY(cudaMemsetAsync(p->d_ut, 0, sizeof(double) * (size_t)p->h_ut_off[L], st));
    return OSPH_OK;
  }
  // windows in descending m, each within the budget
  const double wbudget = budget_b / 8.0;
  p->windows.clear();
  int m_hi = own_hi;
  while (m_hi >= own_lo) {
    int m_lo = m_hi;
    double acc = (double)order_doubles(L, m_hi, rf);
    while (m_lo > own_lo && acc + (double)order_doubles(L, m_lo - 1, rf) <= wbudget)
      acc += (double)order_doubles(L, --m_lo, rf);
    FwdWindow w;
    w.m_lo = m_lo;
    w.m_hi = m_hi;
    p->windows.push_back(w);
    m_hi = m_lo - 1;
  }
  int64_t mx[4] = {0, 0, 0, 0};
  int max_orders = 1;
  for (FwdWindow& w : p->windows) {
    range_offsets(L, w.m_lo, w.m_hi, ao, xo, po, bo, tot);
    for (int i = 0; i < 4; ++i) mx[i] = std::max(mx[i], tot[i]);
    max_orders = std::max(max_orders, w.m_hi - w.m_lo + 1);
    W_TRY(cudaMalloc(&w.d_offs, sizeof(int64_t) * 4 * (L + 1)));
    W_TRY(cudaMemcpy(w.d_offs, ao.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice));
    W_TRY(cudaMemcpy(w.d_offs + (L + 1), xo.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice));
    W_TRY(cudaMemcpy(w.d_offs + 2 * (L + 1), po.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice));
    W_TRY(cudaMemcpy(w.d_offs + 3 * (L + 1), bo.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice));
    if (bf_prepare(p, w.m_lo, w.m_hi, &w.bf) != cudaSuccess) {
      osph_set_error("window work tables");
      return OSPH_ERR_CUDA;
    }
    for (cudaEvent_t& e : w.ev) W_TRY(cudaEventCreate(&e));
  }
  W_TRY(dalloc_w(&p->d_ainv, (size_t)mx[0]));
  W_TRY(dalloc_w(&p->d_xt, (size_t)mx[1]));
  if (rf) W_TRY(dalloc_w(&p->d_at, (size_t)mx[1]));
  W_TRY(dalloc_w(&p->d_pbelow, (size_t)mx[2]));
  W_TRY(dalloc_w(&p->d_bf_e, (size_t)mx[3]));
  W_TRY(dalloc_w(&p->d_bf_e2, (size_t)mx[3]));
  W_TRY(dalloc_w(&p->d_bf_r, (size_t)(2 * mx[3])));
  W_TRY(cudaMemsetAsync(p->d_bf_r, 0, sizeof(double) * (size_t)(2 * mx[3]), st));
  p->bf_r_half = mx[3];
  W_TRY(dalloc_w(&p->d_bf_d, (size_t)bf_diag_doubles(max_orders)));
  return OSPH_OK;
}

void free_windows(osph_plan* p) {
  for (FwdWindow& w : p->windows) {
    cudaFree(w.d_offs);
    cudaFree(w.bf.d_tab);
    for (cudaEvent_t& e : w.ev)
      if (e) cudaEventDestroy(e);
  }
  p->windows.clear();
  cudaFree(p->bf_full.d_tab);
  p->bf_full.d_tab = nullptr;
}

// Factor + sweep of every window on the plan stream (the right-hand sides R
// are already in place); zero-fills the norms/status first like launch_factor.
cudaError_t forward_windows(osph_plan* p, int B, double2* flm) {
  const int L = p->L;
  cudaStream_t st = p->stream;
  cudaError_t e;
  if ((e = cudaMemsetAsync(p->d_norms, 0, sizeof(unsigned long long) * 2 * L, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p->d_status, 0, sizeof(int) * L, st)) != cudaSuccess) return e;
  for (FwdWindow& w : p->windows) {
    const BfOffsets o{w.d_offs, w.d_offs + (L + 1), w.d_offs + 2 * (L + 1), w.d_offs + 3 * (L + 1)};
    if ((e = cudaEventRecord(w.ev[0], st)) != cudaSuccess) return e;
    if ((e = bf_run(p, w.bf, st, o)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(w.ev[1], st)) != cudaSuccess) return e;
    if ((e = launch_sweep_large_range(p, B, flm, w.m_hi, w.m_lo, o.xt, o.pb)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(w.ev[2], st)) != cudaSuccess) return e;
  }
  return launch_kappa(p, st);
}

// Staged windowed forward (sharded plans, osph_forward_stage): the first
// window's factorisation alone (it reads no data, so it can run before the
// right-hand sides arrive from the previous shard), then the sweep of every
// window with windows >= 1 factored just before their sweep (they reuse the
// storage of the window before).
cudaError_t forward_windows_factor_first(osph_plan* p) {
  const int L = p->L;
  cudaStream_t st = p->stream;
  cudaError_t e;
  if ((e = cudaMemsetAsync(p->d_norms, 0, sizeof(unsigned long long) * 2 * L, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p->d_status, 0, sizeof(int) * L, st)) != cudaSuccess) return e;
  if (p->windows.empty()) return cudaSuccess;
  FwdWindow& w = p->windows[0];
  const BfOffsets o{w.d_offs, w.d_offs + (L + 1), w.d_offs + 2 * (L + 1), w.d_offs + 3 * (L + 1)};
  if ((e = cudaEventRecord(w.ev[0], st)) != cudaSuccess) return e;
  if ((e = bf_run(p, w.bf, st, o)) != cudaSuccess) return e;
  return cudaEventRecord(w.ev[1], st);
}

cudaError_t forward_windows_sweep(osph_plan* p, int B, double2* flm) {
  const int L = p->L;
  cudaStream_t st = p->stream;
  cudaError_t e;
  for (size_t i = 0; i < p->windows.size(); ++i) {
    FwdWindow& w = p->windows[i];
    const BfOffsets o{w.d_offs, w.d_offs + (L + 1), w.d_offs + 2 * (L + 1), w.d_offs + 3 * (L + 1)};
    if (i > 0) {
      if ((e = cudaEventRecord(w.ev[0], st)) != cudaSuccess) return e;
      if ((e = bf_run(p, w.bf, st, o)) != cudaSuccess) return e;
      if ((e = cudaEventRecord(w.ev[1], st)) != cudaSuccess) return e;
    }
    if ((e = launch_sweep_large_range(p, B, flm, w.m_hi, w.m_lo, o.xt, o.pb)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(w.ev[2], st)) != cudaSuccess) return e;
  }
  return launch_kappa(p, st);
}

// Device milliseconds of the last windowed forward: factor and sweep summed over windows.
void window_times(osph_plan* p) {
  float f = 0.f, s = 0.f;
  for (FwdWindow& w : p->windows) {
    float a = 0.f, b = 0.f;
    cudaEventSynchronize(w.ev[2]);
    cudaEventElapsedTime(&a, w.ev[0], w.ev[1]);
    cudaEventElapsedTime(&b, w.ev[1], w.ev[2]);
    f += a;
    s += b;
  }
  p->last_factor_ms = f;
  p->last_sweep_ms = s;
}
