// plan.cu -- C ABI of libosph (include/osph.h): plan life cycle and the
// forward / inverse transform pipelines.
//
//   osph_inverse = inverse_sht   (pkg/src/optisph/transform.py:347-357):
//       pack (flm -> per-order columns) -> synth (Legendre sums, G) ->
//       ring inverse DFTs (fold + Bluestein)
//   osph_forward = forward_sht   (transform.py:360-467, spectral method):
//       ring forward DFTs -> per-order factorisation (data independent) ->
//       order-peeling sweep
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#include "../../include/osph.h"
#include "plan.cuh"

static thread_local std::string g_last_error;

void osph_set_error(const std::string& msg) { g_last_error = msg; }

void plan_dft_layout(osph_plan* p, std::vector<int>& bluestein_rings);  // tables.cu

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) {                                                                  \
      osph_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                     \
      return OSPH_ERR_CUDA;                                                                   \
    }                                                                                         \
  } while (0)

template <typename T>
static cudaError_t dalloc(T** ptr, size_t count) {
  return cudaMalloc(reinterpret_cast<void**>(ptr), sizeof(T) * std::max<size_t>(count, 1));
}

template <typename T>
static cudaError_t upload(T** ptr, const T* host, size_t count, cudaStream_t st) {
  cudaError_t e = dalloc(ptr, count);
  if (e != cudaSuccess) return e;
  if (count) e = cudaMemcpyAsync(*ptr, host, sizeof(T) * count, cudaMemcpyHostToDevice, st);
  return e;
}

void plan_free(osph_plan* p) {
  if (!p) return;
  for (osph_plan* q : p->group) plan_free(q);
  for (osph_plan* q : p->group_maps) plan_free(q);
  cudaSetDevice(p->device);
  void* ptrs[] = {p->d_cos, p->d_sin, p->d_rec, p->d_ls, p->d_pstart, p->d_ring_order, p->d_fft_n,
                  p->d_chirp_off, p->d_bhat_off, p->d_chirp, p->d_bhat, p->d_tw, p->d_roots,
                  p->d_bluestein_rings, p->d_ainv_off, p->d_pb_off, p->d_ainv, p->d_pbelow, p->d_piv,
                  p->d_norms, p->d_kappa, p->d_status, p->d_jstar, p->d_beta, p->d_u, p->d_w, p->d_xt_off, p->d_xt,
                  p->d_fpack, p->d_g, p->d_r,
                  p->d_in, p->d_out, p->d_sw, p->d_rtw, p->d_ut_off, p->d_ut, p->d_sb_x, p->d_sb_a, p->d_sb_g, p->d_sb_r2, p->d_xbuf, p->d_rres, p->d_at, p->d_bf_off, p->d_bf_e, p->d_bf_e2, p->d_bf_r,
                  p->d_bf_d};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  for (cudaEvent_t& e : p->ev)
    if (e) cudaEventDestroy(e);
  for (int c = 0; c < osph_plan::kIoChunks; ++c) {
    if (p->ev_in[c]) cudaEventDestroy(p->ev_in[c]);
    if (p->ev_done[c]) cudaEventDestroy(p->ev_done[c]);
  }
  if (p->ev_start) cudaEventDestroy(p->ev_start);
  if (p->ev_out) cudaEventDestroy(p->ev_out);
  if (p->ev_sweep_done) cudaEventDestroy(p->ev_sweep_done);
  if (p->s_in) cudaStreamDestroy(p->s_in);
  for (int r = 0; r < osph_plan::kFactorRanges; ++r) {
    if (p->s_f[r]) cudaStreamDestroy(p->s_f[r]);
    if (p->ev_f[r]) cudaEventDestroy(p->ev_f[r]);
    cudaFree(p->bf_rng[r].d_tab);
  }
  if (p->ev_fstart) cudaEventDestroy(p->ev_fstart);
  cudaFree(p->bf_full.d_tab);
  if (p->s_out) cudaStreamDestroy(p->s_out);
  cudaFree(p->d_z1);
  cudaFree(p->d_z2);
  if (p->inv_own_lists) {
    cudaFree(p->d_inv_ring_order);
    cudaFree(p->d_inv_bluestein);
  }
  free_windows(p);
  spin_free(p);
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

extern "C" int osph_abi_version(void) { return OSPH_ABI_VERSION; }

extern "C" const char* osph_last_error(void) { return g_last_error.c_str(); }

extern "C" int osph_plan_create(int L, const double* thetas, int max_batch, int ndev, const int* devs,
                                osph_plan** out) {
  DeviceGuard guard;
  g_last_error.clear();
  if (out) *out = nullptr;
  if (ndev < 1 || !devs) {
    osph_set_error("osph_plan_create: ndev must be >= 1 with a device list");
    return OSPH_ERR_ARG;
  }
  if (ndev > 1) return group_create(L, thetas, max_batch, ndev, devs, out);
  return plan_create_one(L, thetas, max_batch, devs[0], out);
}

int plan_create_one(int L, const double* thetas, int max_batch, int device, osph_plan** out) {
  if (!out) {
    osph_set_error("osph_plan_create: out is NULL");
    return OSPH_ERR_ARG;
  }
  *out = nullptr;
  if (L < 1 || L > 4096) {
    osph_set_error("band limit must be in [1, 4096], got " + std::to_string(L));
    return OSPH_ERR_ARG;
  }
  if (max_batch < 1) {
    osph_set_error("max_batch must be positive");
    return OSPH_ERR_ARG;
  }
  if (!thetas) {
    osph_set_error("thetas is NULL");
    return OSPH_ERR_ARG;
  }
  for (int k = 0; k < L; ++k) {
    if (!(thetas[k] > 0.0 && thetas[k] <= OSPH_PI)) {  // ColatitudeGrid invariant (sampling.py:69-70)
      osph_set_error("co-latitudes must lie in (0, pi]");
      return OSPH_ERR_ARG;
    }
  }
  int ndev = 0;
  cudaError_t e0 = cudaGetDeviceCount(&ndev);
  if (e0 != cudaSuccess || ndev == 0) {
    osph_set_error(std::string("no CUDA device available: ") + cudaGetErrorString(e0));
    return OSPH_ERR_CUDA;
  }
  if (device < 0 || device >= ndev) {
    osph_set_error("device ordinal out of range");
    return OSPH_ERR_ARG;
  }
  osph_plan* p = new osph_plan();
  p->L = L;
  p->device = device;
  p->max_batch = max_batch;
  auto fail = [&](int code) {
    plan_free(p);
    return code;
  };
#define PLAN_TRY(expr)                                                    \
  do {                                                                    \
    cudaError_t _e = (expr);                                              \
    if (_e != cudaSuccess) {                                              \
      osph_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
      return fail(OSPH_ERR_CUDA);                                         \
    }                                                                     \
  } while (0)
  PLAN_TRY(cudaSetDevice(device));
  PLAN_TRY(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  p->own_stream = true;
  for (cudaEvent_t& e : p->ev) PLAN_TRY(cudaEventCreate(&e));
  // the factorisation streams run at the highest priority: the factor is the
  // critical path into the sweep, the work beside it (inverse, ring DFTs) is not
  int prio_lo = 0, prio_hi = 0;
  PLAN_TRY(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  if (getenv("OSPH_NO_STREAM_PRIORITY")) prio_hi = prio_lo;
  PLAN_TRY(cudaStreamCreateWithPriority(&p->s_in, cudaStreamNonBlocking, prio_hi));
  PLAN_TRY(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
  for (int r = 0; r < osph_plan::kFactorRanges - 1; ++r) {
    PLAN_TRY(cudaStreamCreateWithPriority(&p->s_f[r], cudaStreamNonBlocking, prio_hi));
    PLAN_TRY(cudaEventCreateWithFlags(&p->ev_f[r], cudaEventDisableTiming));
  }
  PLAN_TRY(cudaEventCreateWithFlags(&p->ev_fstart, cudaEventDisableTiming));
  for (int c = 0; c < osph_plan::kIoChunks; ++c) {
    PLAN_TRY(cudaEventCreateWithFlags(&p->ev_in[c], cudaEventDisableTiming));
    PLAN_TRY(cudaEventCreateWithFlags(&p->ev_done[c], cudaEventDisableTiming));
  }
  PLAN_TRY(cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming));
  PLAN_TRY(cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming));
  PLAN_TRY(cudaEventCreateWithFlags(&p->ev_sweep_done, cudaEventDisableTiming));
  cudaStream_t st = p->stream;

  p->h_thetas.assign(thetas, thetas + L);
  std::vector<double> c(L), s(L);
  for (int k = 0; k < L; ++k) {
    c[k] = std::cos(thetas[k]);
    s[k] = std::sin(thetas[k]);
  }
  PLAN_TRY(upload(&p->d_cos, c.data(), L, st));
  PLAN_TRY(upload(&p->d_sin, s.data(), L, st));
  std::vector<int> order(L);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return s[a] < s[b]; });
  PLAN_TRY(upload(&p->d_ring_order, order.data(), L, st));
  p->h_ring_order = order;
  const size_t npacked = (size_t)L * (L + 1) / 2;
  PLAN_TRY(dalloc(&p->d_rec, npacked));
  PLAN_TRY(dalloc(&p->d_ls, (size_t)L * L));
  PLAN_TRY(dalloc(&p->d_pstart, (size_t)L * L));

  std::vector<int> brings;
  plan_dft_layout(p, brings);
  PLAN_TRY(upload(&p->d_fft_n, p->h_fft_n.data(), L, st));
  PLAN_TRY(upload(&p->d_chirp_off, p->h_chirp_off.data(), L, st));
  PLAN_TRY(upload(&p->d_bhat_off, p->h_bhat_off.data(), L, st));
  PLAN_TRY(upload(&p->d_bluestein_rings, brings.data(), brings.size(), st));
  p->h_bluestein_rings = brings;
  PLAN_TRY(dalloc(&p->d_chirp, (size_t)p->h_chirp_off[L]));
  PLAN_TRY(dalloc(&p->d_bhat, (size_t)p->h_bhat_off[L]));
  PLAN_TRY(dalloc(&p->d_tw, 8192));
  PLAN_TRY(dalloc(&p->d_roots, (size_t)(OSPH_DIRECT_MAX + 1) * (OSPH_DIRECT_MAX + 1) / 4 + 64));
  PLAN_TRY(dalloc(&p->d_sw, OSPH_SW_GLOBAL));
  PLAN_TRY(dalloc(&p->d_rtw, OSPH_RTW_SIZE));
  // OSPH_RING_REG=0: every Bluestein ring on the shared-memory transforms of fft.cuh (A/B measurements)
  p->reg_fft_max = (getenv("OSPH_RING_REG") && atoi(getenv("OSPH_RING_REG")) == 0) ? 0 : OSPH_REG_FFT_MAX;
  for (int k = 0; k < L; ++k) {
    if (p->h_fft_n[k] > 2 * OSPH_FFT_MAX) p->dft_ok = false;
    if (p->h_fft_n[k] > OSPH_FFT_MAX) p->n_big_rings++;
  }
  if (!p->dft_ok) p->n_bluestein_rings = p->n_big_rings = 0;  // Legendre tables only (osph_legendre_block)
  for (int k : brings)
    if (p->dft_ok && p->h_fft_n[k] <= p->reg_fft_max) {
      p->n_reg_rings++;
      if (p->h_fft_n[k] == 2048) p->n_reg2_rings++;
    }
  // the inverse produces every ring until osph_plan_shard restricts it
  p->inv_nr = L;
  p->d_inv_ring_order = p->d_ring_order;
  p->d_inv_bluestein = p->d_bluestein_rings;
  p->inv_n_bluestein = p->n_bluestein_rings;
  p->inv_n_big = p->n_big_rings;
  p->inv_n_reg = p->n_reg_rings;
  p->inv_n_reg2 = p->n_reg2_rings;
  p->inv_direct_lo = 0;
  p->inv_direct_hi = p->n_direct_rings;
  p->own_k_lo = 0;
  p->own_k_hi = L;
  PLAN_TRY(launch_tables(p));
  PLAN_TRY(cudaStreamSynchronize(st));
  *out = p;
  return OSPH_OK;
#undef PLAN_TRY
}

extern "C" int osph_plan_destroy(osph_plan* plan) {
  DeviceGuard guard;
  plan_free(plan);
  return OSPH_OK;
}

extern "C" int osph_plan_set_stream(osph_plan* p, void* stream) {
  DeviceGuard guard;
  if (!p) {
    osph_set_error("plan is NULL");
    return OSPH_ERR_ARG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  if (!stream && p->own_stream) return OSPH_OK;  // already on a plan-owned stream
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
  p->own_stream = false;
  p->stream = (cudaStream_t)stream;
  if (!stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    p->own_stream = true;
  }
  return OSPH_OK;
}

extern "C" int osph_plan_info(const osph_plan* p, int* L, int* max_batch) {
  if (!p) {
    osph_set_error("plan is NULL");
    return OSPH_ERR_ARG;
  }
  if (L) *L = p->L;
  if (max_batch) *max_batch = p->max_batch;
  return OSPH_OK;
}

extern "C" int osph_last_launch_count(const osph_plan* p) { return p ? p->launches : 0; }

int ensure_io(osph_plan* p) {
  if (p->d_in) return OSPH_OK;
  const size_t n = (size_t)p->max_batch * p->L * p->L;
  CUDA_TRY(dalloc(&p->d_in, n));
  CUDA_TRY(dalloc(&p->d_out, n));
  return OSPH_OK;
}

int ensure_inverse(osph_plan* p) {
  if (p->inv_ready) return OSPH_OK;
  const int L = p->L;
  const size_t B = p->max_batch;
  CUDA_TRY(dalloc(&p->d_fpack, (size_t)L * (L + 1) / 2 * 4 * B));
  CUDA_TRY(dalloc(&p->d_g, (size_t)L * L * 4 * B));
  p->inv_ready = true;
  return OSPH_OK;
}

int ensure_forward(osph_plan* p) {
  if (p->fwd_ready) return OSPH_OK;
  const int L = p->L;
  const size_t B = p->max_batch;
  cudaStream_t st = p->stream;
  int rc;
  if ((rc = alloc_factor_storage(p))) return rc;
  CUDA_TRY(dalloc(&p->d_piv, (size_t)L * (L + 1) / 2));
  CUDA_TRY(dalloc(&p->d_norms, (size_t)2 * L));
  CUDA_TRY(dalloc(&p->d_kappa, (size_t)L));
  CUDA_TRY(dalloc(&p->d_status, (size_t)L));
  CUDA_TRY(dalloc(&p->d_jstar, (size_t)L));
  CUDA_TRY(dalloc(&p->d_beta, (size_t)L));
  CUDA_TRY(dalloc(&p->d_xbuf, (size_t)2 * L * B));
  CUDA_TRY(dalloc(&p->d_rres, (size_t)2 * L * B));

  // [L][L] + 2: the sweep's bulk copies round their sizes up to 16 bytes
  const size_t nuw = (size_t)L * uw_ld(L) + 2;  // even row stride: aligned rows for bulk copies
  CUDA_TRY(dalloc(&p->d_u, nuw));
  CUDA_TRY(dalloc(&p->d_w, nuw));
  CUDA_TRY(cudaMemsetAsync(p->d_u, 0, sizeof(double) * nuw, st));
  CUDA_TRY(cudaMemsetAsync(p->d_w, 0, sizeof(double) * nuw, st));
  if ((rc = ensure_spectra(p))) return rc;
  CUDA_TRY(cudaStreamSynchronize(st));
  p->fwd_ready = true;
  return OSPH_OK;
}

// The ring spectra R (teams of up to 4 maps: the last team's padding maps stay zero).
int ensure_spectra(osph_plan* p) {
  if (p->d_r) return OSPH_OK;
  const size_t n = (size_t)p->L * (p->L + 1) * (p->max_batch + 3);
  CUDA_TRY(dalloc(&p->d_r, n));
  CUDA_TRY(cudaMemsetAsync(p->d_r, 0, sizeof(double2) * n, p->stream));
  return OSPH_OK;
}

static int sweep_kind(const osph_plan* p) {
  if (p->windowed) return OSPH_SWEEP_WINDOWED;
  if (p->sweep_blocked) return OSPH_SWEEP_BLOCKED;
  if (p->sweep_gemm) return OSPH_SWEEP_GEMM;
  if (p->sweep_large) return OSPH_SWEEP_LARGE;
  return OSPH_SWEEP_PERSISTENT;
}

int check_call(osph_plan* p, int B, const void* a, void* b, int kind) {
  if (!p) {
    osph_set_error("plan is NULL");
    return OSPH_ERR_ARG;
  }
  if (!p->dft_ok) {
    osph_set_error("ring DFT length exceeds the two-CTA Bluestein FFT (transforms need L <= 4096)");
    return OSPH_ERR_ARG;
  }
  if (B < 1 || B > p->max_batch) {
    osph_set_error("batch " + std::to_string(B) + " outside [1, max_batch=" + std::to_string(p->max_batch) + "]");
    return OSPH_ERR_ARG;
  }
  if (!a || !b) {
    osph_set_error("NULL data pointer");
    return OSPH_ERR_ARG;
  }
  if (kind & ~(OSPH_DEVICE | OSPH_ASYNC | OSPH_REAL)) {
    osph_set_error("unknown ptr_kind flags");
    return OSPH_ERR_ARG;
  }
  if ((kind & OSPH_ASYNC) && !(kind & OSPH_DEVICE)) {
    osph_set_error("OSPH_ASYNC requires OSPH_DEVICE pointers");
    return OSPH_ERR_ARG;
  }
  return OSPH_OK;
}

// Host buffers: the batch is cut into up to kIoChunks map chunks; chunk c's
// H2D copy (s_in), compute (plan stream) and D2H copy (s_out) are chained by
// events, so copies of neighbouring chunks overlap the compute in both
// directions.  Device buffers: one pass on the plan stream.
// ---------------------------------------------------------------------------
// Real maps (OSPH_REAL).  The transforms are complex-linear, so two real maps
// a, b run as ONE complex map z = a + i b: the inverse of f_a + i f_b is
// a + i b (both syntheses are real), and the forward of a + i b is
// F(a) + i F(b) with F(a)_{l,-m} = (-1)^m conj F(a)_{lm}, so
//   F(a)_lm = (z_lm + c) / 2,  F(b)_lm = (z_lm - c) / (2i),  c = (-1)^m conj z_{l,-m}.
// Half the maps go through the transform; pairing/unpairing are one HBM pass each.

__global__ void k_pair_flm(int B, int64_t n, const double2* __restrict__ f, double2* __restrict__ z) {
  const int p = blockIdx.y;
  const double2* fa = f + (size_t)(2 * p) * n;
  const double2* fb = (2 * p + 1 < B) ? f + (size_t)(2 * p + 1) * n : nullptr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = fa[i];
    const double2 b = fb ? fb[i] : make_double2(0.0, 0.0);
    z[(size_t)p * n + i] = make_double2(a.x - b.y, a.y + b.x);
  }
}

__global__ void k_unpair_samples(int B, int64_t n, const double2* __restrict__ z, double2* __restrict__ s) {
  const int p = blockIdx.y;
  double2* sa = s + (size_t)(2 * p) * n;
  double2* sb = (2 * p + 1 < B) ? s + (size_t)(2 * p + 1) * n : nullptr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = z[(size_t)p * n + i];
    sa[i] = make_double2(v.x, 0.0);
    if (sb) sb[i] = make_double2(v.y, 0.0);
  }
}

__global__ void k_pair_samples(int B, int64_t n, const double2* __restrict__ s, double2* __restrict__ z) {
  const int p = blockIdx.y;
  const double2* sa = s + (size_t)(2 * p) * n;
  const double2* sb = (2 * p + 1 < B) ? s + (size_t)(2 * p + 1) * n : nullptr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[(size_t)p * n + i] = make_double2(sa[i].x, sb ? sb[i].x : 0.0);
}

// flm index i = l^2 + l + m; its mirror l^2 + l - m = 2(l^2 + l) - i.
__global__ void k_unpair_flm(int B, int L, const double2* __restrict__ z, double2* __restrict__ f) {
  const int p = blockIdx.y;
  const int64_t n = (int64_t)L * L;
  const double2* zp = z + (size_t)p * n;
  double2* fa = f + (size_t)(2 * p) * n;
  double2* fb = (2 * p + 1 < B) ? f + (size_t)(2 * p + 1) * n : nullptr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = (int64_t)sqrt((double)i);
    const int64_t ll = (l * l > i) ? l - 1 : ((l + 1) * (l + 1) <= i ? l + 1 : l);
    const int64_t c0 = ll * ll + ll;
    const int64_t m = i - c0;
    const double sg = (m & 1) ? -1.0 : 1.0;
    const double2 a = zp[i], b = zp[2 * c0 - i];
    const double2 c = make_double2(sg * b.x, -sg * b.y);  // (-1)^m conj z_{l,-m}
    fa[i] = make_double2(0.5 * (a.x + c.x), 0.5 * (a.y + c.y));
    if (fb) fb[i] = make_double2(0.5 * (a.y - c.y), -0.5 * (a.x - c.x));  // (a - c) / 2i
  }
}

// The sweep on `st` waits for the factorisation, recorded as ev[7] on a side stream.  The
// blocked sweep of a split factorisation (factor.cu) waits range by range instead, each at
// its first block of that range (launch_sweep_blocked; the lowest range's event is ev[7]).
static cudaError_t wait_factor_for_sweep(osph_plan* p, cudaStream_t st) {
  p->sweep_waits_ranges = p->fsplit_active && p->sweep_blocked;
  return p->sweep_waits_ranges ? cudaSuccess : cudaStreamWaitEvent(st, p->ev[7], 0);
}

static int ensure_real(osph_plan* p) {
  if (p->d_z1) return OSPH_OK;
  const size_t n = (size_t)((p->max_batch + 1) / 2) * p->L * p->L;
  CUDA_TRY(dalloc(&p->d_z1, n));
  CUDA_TRY(dalloc(&p->d_z2, n));
  return OSPH_OK;
}

static dim3 pair_grid(int pairs, int64_t n) {
  return dim3((unsigned)std::min<int64_t>((n + 255) / 256, 1184), (unsigned)pairs);
}

// Host buffers, real maps: the batch goes through in chunks of whole pairs -- chunk c's
// H2D copy (s_in), pairing + transform + unpairing (plan stream) and D2H copy (s_out) are
// chained by events, so the copies of neighbouring chunks overlap the kernels in both
// directions (the copies, 2 x 16 B L^2 per real map and direction, bound this path).
static int inverse_real_host_chunked(osph_plan* p, int B, const void* flm, void* samples) {
  const int L = p->L;
  const int64_t n = (int64_t)L * L;
  cudaStream_t st = p->stream;
  const int npairs = (B + 1) / 2, nch = std::min(npairs, osph_plan::kIoChunks);
  CUDA_TRY(cudaEventRecord(p->ev_start, st));
  CUDA_TRY(cudaStreamWaitEvent(p->s_in, p->ev_start, 0));
  CUDA_TRY(cudaStreamWaitEvent(p->s_out, p->ev_start, 0));
  for (int c = 0; c < nch; ++c) {
    const int q0 = (int)((int64_t)npairs * c / nch), q1 = (int)((int64_t)npairs * (c + 1) / nch);  // pairs
    const int b0 = 2 * q0, b1 = std::min(B, 2 * q1), bc = b1 - b0, qc = q1 - q0;
    const size_t off = (size_t)b0 * n, zoff = (size_t)q0 * n, cb = sizeof(double2) * (size_t)bc * n;
    CUDA_TRY(cudaMemcpyAsync(p->d_in + off, (const double2*)flm + off, cb, cudaMemcpyHostToDevice, p->s_in));
    CUDA_TRY(cudaEventRecord(p->ev_in[c], p->s_in));
    CUDA_TRY(cudaStreamWaitEvent(st, p->ev_in[c], 0));
    k_pair_flm<<<pair_grid(qc, n), 256, 0, st>>>(bc, n, p->d_in + off, p->d_z1 + zoff);
    if (c == 0) CUDA_TRY(cudaEventRecord(p->ev[0], st));
    CUDA_TRY(launch_pack(p, qc, p->d_z1 + zoff));
    if (c == 0) CUDA_TRY(cudaEventRecord(p->ev[1], st));
    CUDA_TRY(launch_synth(p, qc));
    if (c == 0) CUDA_TRY(cudaEventRecord(p->ev[2], st));
    CUDA_TRY(launch_ring_inverse(p, qc, p->d_z2 + zoff));
    k_unpair_samples<<<pair_grid(qc, n), 256, 0, st>>>(bc, n, p->d_z2 + zoff, p->d_out + off);
    CUDA_TRY(cudaGetLastError());
    p->launches += 2;
    CUDA_TRY(cudaEventRecord(p->ev_done[c], st));
    CUDA_TRY(cudaStreamWaitEvent(p->s_out, p->ev_done[c], 0));
    CUDA_TRY(cudaMemcpyAsync((double2*)samples + off, p->d_out + off, cb, cudaMemcpyDeviceToHost, p->s_out));
  }
  CUDA_TRY(cudaEventRecord(p->ev[3], st));
  CUDA_TRY(cudaEventRecord(p->ev_out, p->s_out));
  CUDA_TRY(cudaStreamWaitEvent(st, p->ev_out, 0));  // the plan stream covers the whole call
  return OSPH_OK;
}

static int inverse_real(osph_plan* p, int B, const void* flm, void* samples, bool host) {
  int rc;
  if ((rc = ensure_real(p))) return rc;
  if (host && p->own_k_lo == 0 && p->own_k_hi == p->L) return inverse_real_host_chunked(p, B, flm, samples);
  const int L = p->L, Bp = (B + 1) / 2;
  const int64_t n = (int64_t)L * L;
  const size_t bytes = sizeof(double2) * (size_t)B * n;
  cudaStream_t st = p->stream;
  const double2* src = (const double2*)flm;
  double2* dst = (double2*)samples;
  if (host) {
    CUDA_TRY(cudaMemcpyAsync(p->d_in, flm, bytes, cudaMemcpyHostToDevice, st));
    src = p->d_in;
    dst = p->d_out;
  }
  k_pair_flm<<<pair_grid(Bp, n), 256, 0, st>>>(B, n, src, p->d_z1);
  CUDA_TRY(cudaEventRecord(p->ev[0], st));
  CUDA_TRY(launch_pack(p, Bp, p->d_z1));
  CUDA_TRY(cudaEventRecord(p->ev[1], st));
  CUDA_TRY(launch_synth(p, Bp));
  CUDA_TRY(cudaEventRecord(p->ev[2], st));
  CUDA_TRY(launch_ring_inverse(p, Bp, p->d_z2));
  CUDA_TRY(cudaEventRecord(p->ev[3], st));
  k_unpair_samples<<<pair_grid(Bp, n), 256, 0, st>>>(B, n, p->d_z2, dst);
  CUDA_TRY(cudaGetLastError());
  p->launches += 2;
  if (host) CUDA_TRY(cudaMemcpyAsync(samples, p->d_out, bytes, cudaMemcpyDeviceToHost, st));
  return OSPH_OK;
}

// Host buffers, real maps, blocked sweep: chunks of whole pairs are copied in (s_in) while the
// factorisation runs; each chunk is paired and ring-transformed as it lands; the batch is
// swept, unpaired and copied out (s_out) in two halves, so the first half's coefficients cross
// PCIe while the second half is swept.
static int forward_real_host_chunked(osph_plan* p, int B, const void* samples, void* flm) {
  const int L = p->L;
  const int64_t n = (int64_t)L * L;
  cudaStream_t st = p->stream;
  const int npairs = (B + 1) / 2, nch = osph_plan::kIoChunks;
  CUDA_TRY(cudaEventRecord(p->ev_start, st));
  CUDA_TRY(cudaStreamWaitEvent(p->s_in, p->ev_start, 0));
  CUDA_TRY(cudaStreamWaitEvent(p->s_out, p->ev_start, 0));
  for (int c = 0; c < nch; ++c) {
    const int q0 = (int)((int64_t)npairs * c / nch), q1 = (int)((int64_t)npairs * (c + 1) / nch);
    const int b0 = 2 * q0, b1 = std::min(B, 2 * q1);
    const size_t off = (size_t)b0 * n, cb = sizeof(double2) * (size_t)(b1 - b0) * n;
    CUDA_TRY(cudaMemcpyAsync(p->d_in + off, (const double2*)samples + off, cb, cudaMemcpyHostToDevice, p->s_in));
    CUDA_TRY(cudaEventRecord(p->ev_in[c], p->s_in));
  }
  CUDA_TRY(cudaEventRecord(p->ev[6], st));
  CUDA_TRY(launch_factor(p, st));
  CUDA_TRY(cudaEventRecord(p->ev[7], st));
  for (int c = 0; c < nch; ++c) {
    const int q0 = (int)((int64_t)npairs * c / nch), q1 = (int)((int64_t)npairs * (c + 1) / nch);
    const int b0 = 2 * q0, b1 = std::min(B, 2 * q1), bc = b1 - b0, qc = q1 - q0;
    const size_t off = (size_t)b0 * n, zoff = (size_t)q0 * n;
    CUDA_TRY(cudaStreamWaitEvent(st, p->ev_in[c], 0));
    k_pair_samples<<<pair_grid(qc, n), 256, 0, st>>>(bc, n, p->d_in + off, p->d_z1 + zoff);
    p->launches++;
    if (c == 0) CUDA_TRY(cudaEventRecord(p->ev[4], st));
    CUDA_TRY(launch_ring_forward(p, npairs, p->d_z1, q0, qc));
    if (c == nch / 2 - 1 || c == nch - 1) {
      const int h = c == nch - 1;
      const int hq0 = h ? (int)((int64_t)npairs * (nch / 2) / nch) : 0, hq1 = h ? npairs : (int)((int64_t)npairs * (nch / 2) / nch);
      const int hb0 = 2 * hq0, hb1 = std::min(B, 2 * hq1);
      const size_t hoff = (size_t)hb0 * n, hz = (size_t)hq0 * n, hbytes = sizeof(double2) * (size_t)(hb1 - hb0) * n;
      if (h == 0) CUDA_TRY(cudaEventRecord(p->ev[8], st));
      CUDA_TRY(launch_sweep_blocked(p, hq1 - hq0, p->d_z2 + hz, hq0));
      k_unpair_flm<<<pair_grid(hq1 - hq0, n), 256, 0, st>>>(hb1 - hb0, L, p->d_z2 + hz, p->d_out + hoff);
      CUDA_TRY(cudaGetLastError());
      p->launches++;
      CUDA_TRY(cudaEventRecord(p->ev_done[h], st));
      CUDA_TRY(cudaStreamWaitEvent(p->s_out, p->ev_done[h], 0));
      CUDA_TRY(cudaMemcpyAsync((double2*)flm + hoff, p->d_out + hoff, hbytes, cudaMemcpyDeviceToHost, p->s_out));
    }
  }
  CUDA_TRY(cudaEventRecord(p->ev[5], st));
  p->last_sweep_kind = OSPH_SWEEP_BLOCKED;
  CUDA_TRY(cudaEventRecord(p->ev[9], st));
  CUDA_TRY(cudaEventRecord(p->ev_sweep_done, st));
  p->have_sweep_ev = true;
  CUDA_TRY(cudaEventRecord(p->ev_out, p->s_out));
  CUDA_TRY(cudaStreamWaitEvent(st, p->ev_out, 0));
  return OSPH_OK;
}

static int forward_real(osph_plan* p, int B, const void* samples, void* flm, bool host) {
  int rc;
  if ((rc = ensure_real(p))) return rc;
  if (host && !p->windowed && (B + 1) / 2 >= 4 * osph_plan::kIoChunks) {
    sweep_maps_per_team(p, (B + 1) / 2);  // decides the sweep (and the layout of the spectra)
    if (p->sweep_blocked && !ensure_sweep_blocked(p)) return forward_real_host_chunked(p, B, samples, flm);
  }
  const int L = p->L, Bp = (B + 1) / 2;
  const int64_t n = (int64_t)L * L;
  const size_t bytes = sizeof(double2) * (size_t)B * n;
  cudaStream_t st = p->stream;
  const double2* src = (const double2*)samples;
  double2* dst = (double2*)flm;
  // the factorisation needs no data: side streams, beside the copy, pairing and ring DFTs
  // (it waits only for the previous forward's sweep, see osph_forward)
  if (p->have_sweep_ev && !p->windowed) {
    CUDA_TRY(cudaStreamWaitEvent(p->s_in, p->ev_sweep_done, 0));
  } else {
    CUDA_TRY(cudaEventRecord(p->ev_start, st));
    CUDA_TRY(cudaStreamWaitEvent(p->s_in, p->ev_start, 0));
  }
  CUDA_TRY(cudaEventRecord(p->ev[6], p->s_in));
  if (!p->windowed) CUDA_TRY(launch_factor(p, p->s_in));
  CUDA_TRY(cudaEventRecord(p->ev[7], p->s_in));
  if (host) {
    CUDA_TRY(cudaMemcpyAsync(p->d_in, samples, bytes, cudaMemcpyHostToDevice, st));
    src = p->d_in;
    dst = p->d_out;
  }
  k_pair_samples<<<pair_grid(Bp, n), 256, 0, st>>>(B, n, src, p->d_z1);
  CUDA_TRY(cudaEventRecord(p->ev[4], st));
  CUDA_TRY(launch_ring_forward(p, Bp, p->d_z1));
  CUDA_TRY(cudaEventRecord(p->ev[5], st));
  if (p->windowed) CUDA_TRY(cudaStreamWaitEvent(st, p->ev[7], 0));
  else CUDA_TRY(wait_factor_for_sweep(p, st));
  CUDA_TRY(cudaEventRecord(p->ev[8], st));
  if (p->windowed) CUDA_TRY(forward_windows(p, Bp, p->d_z2));
  else CUDA_TRY(launch_sweep(p, Bp, p->d_z2));
  p->last_sweep_kind = sweep_kind(p);
  CUDA_TRY(cudaEventRecord(p->ev[9], st));
  CUDA_TRY(cudaEventRecord(p->ev_sweep_done, st));
  p->have_sweep_ev = true;
  k_unpair_flm<<<pair_grid(Bp, n), 256, 0, st>>>(B, L, p->d_z2, dst);
  CUDA_TRY(cudaGetLastError());
  p->launches += 2;
  if (host) CUDA_TRY(cudaMemcpyAsync(flm, p->d_out, bytes, cudaMemcpyDeviceToHost, st));
  return OSPH_OK;
}

// Device -> host copy of the rings the plan's inverse produced (every ring, or a
// chain shard's range [own_k_lo, own_k_hi): samples k^2 .. own_k_hi^2 of each map).
static cudaError_t copy_rings_d2h(const osph_plan* p, double2* host, const double2* dev, int nmaps, cudaStream_t st) {
  const size_t per_map = (size_t)p->L * p->L;
  if (p->own_k_lo == 0 && p->own_k_hi == p->L)
    return cudaMemcpyAsync(host, dev, sizeof(double2) * per_map * nmaps, cudaMemcpyDeviceToHost, st);
  const size_t s0 = (size_t)p->own_k_lo * p->own_k_lo, s1 = (size_t)p->own_k_hi * p->own_k_hi;
  if (s1 == s0) return cudaSuccess;
  return cudaMemcpy2DAsync(host + s0, sizeof(double2) * per_map, dev + s0, sizeof(double2) * per_map,
                           sizeof(double2) * (s1 - s0), nmaps, cudaMemcpyDeviceToHost, st);
}

extern "C" int osph_inverse(osph_plan* p, int B, const void* flm, void* samples, int kind) {
  DeviceGuard guard;
  g_last_error.clear();
  if (p && !p->group_devs.empty()) return group_inverse(p, B, flm, samples, kind);
  int rc = inverse_enqueue(p, B, flm, samples, kind);
  if (rc) return rc;
  if (!(kind & OSPH_ASYNC)) CUDA_TRY(cudaStreamSynchronize(p->stream));
  return OSPH_OK;
}

// osph_inverse without the final synchronisation (multi-device plans enqueue every device first).
int inverse_enqueue(osph_plan* p, int B, const void* flm, void* samples, int kind) {
  int rc = check_call(p, B, flm, samples, kind);
  if (rc) return rc;
  if ((kind & OSPH_REAL) && p->shard_mode == OSPH_SHARD_CHAIN) {
    osph_set_error("real-map pairing (OSPH_REAL) is not available on chain-sharded plans");
    return OSPH_ERR_ARG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  if ((rc = ensure_inverse(p))) return rc;
  const bool host = !(kind & OSPH_DEVICE);
  if (host && (rc = ensure_io(p))) return rc;
  const size_t per_map = (size_t)p->L * p->L;
  cudaStream_t st = p->stream;
  p->launches = 0;
  if (kind & OSPH_REAL) {
    if ((rc = inverse_real(p, B, flm, samples, host))) return rc;
  } else if (!host) {
    CUDA_TRY(cudaEventRecord(p->ev[0], st));
    CUDA_TRY(launch_pack(p, B, (const double2*)flm));
    CUDA_TRY(cudaEventRecord(p->ev[1], st));
    CUDA_TRY(launch_synth(p, B));
    CUDA_TRY(cudaEventRecord(p->ev[2], st));
    CUDA_TRY(launch_ring_inverse(p, B, (double2*)samples));
    CUDA_TRY(cudaEventRecord(p->ev[3], st));
  } else {
    const int nch = std::min(B, osph_plan::kIoChunks);
    CUDA_TRY(cudaEventRecord(p->ev_start, st));  // earlier work on the plan stream (staging buffers)
    CUDA_TRY(cudaStreamWaitEvent(p->s_in, p->ev_start, 0));
    CUDA_TRY(cudaStreamWaitEvent(p->s_out, p->ev_start, 0));
    for (int c = 0; c < nch; ++c) {
      const int b0 = (int)((int64_t)B * c / nch), b1 = (int)((int64_t)B * (c + 1) / nch), bc = b1 - b0;
      const size_t off = (size_t)b0 * per_map, bytes = sizeof(double2) * (size_t)bc * per_map;
      CUDA_TRY(cudaMemcpyAsync(p->d_in + off, (const double2*)flm + off, bytes, cudaMemcpyHostToDevice, p->s_in));
      CUDA_TRY(cudaEventRecord(p->ev_in[c], p->s_in));
      CUDA_TRY(cudaStreamWaitEvent(st, p->ev_in[c], 0));
      if (c == 0) CUDA_TRY(cudaEventRecord(p->ev[0], st));
      CUDA_TRY(launch_pack(p, bc, p->d_in + off));
      if (c == 0) CUDA_TRY(cudaEventRecord(p->ev[1], st));
      CUDA_TRY(launch_synth(p, bc));
      if (c == 0) CUDA_TRY(cudaEventRecord(p->ev[2], st));
      CUDA_TRY(launch_ring_inverse(p, bc, p->d_out + off));
      CUDA_TRY(cudaEventRecord(p->ev_done[c], st));
      CUDA_TRY(cudaStreamWaitEvent(p->s_out, p->ev_done[c], 0));
      CUDA_TRY(copy_rings_d2h(p, (double2*)samples + off, p->d_out + off, bc, p->s_out));
    }
    CUDA_TRY(cudaEventRecord(p->ev[3], st));
    CUDA_TRY(cudaEventRecord(p->ev_out, p->s_out));
    CUDA_TRY(cudaStreamWaitEvent(st, p->ev_out, 0));  // the plan stream covers the whole call
  }
  p->have_inv = true;
  return OSPH_OK;
}

extern "C" int osph_forward(osph_plan* p, int B, const void* samples, void* flm, int kind, int check,
                            osph_stats* stats) {
  DeviceGuard guard;
  g_last_error.clear();
  if (p && !p->group_devs.empty()) return group_forward(p, B, samples, flm, kind, check, stats);
  int rc = check_call(p, B, samples, flm, kind);
  if (rc) return rc;
  if (p->shard_mode) {
    osph_set_error("a sharded plan runs the forward in stages (osph_forward_stage)");
    return OSPH_ERR_ARG;
  }
  if ((kind & OSPH_ASYNC) && check) {
    osph_set_error("check=1 needs a host-blocking call (drop OSPH_ASYNC or pass check=0)");
    return OSPH_ERR_ARG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  if ((rc = ensure_forward(p))) return rc;
  if (!p->piv_ready && (rc = discover_pivots(p))) return rc;
  p->need_norms = check != 0;
  const bool host = !(kind & OSPH_DEVICE);
  if (host && (rc = ensure_io(p))) return rc;
  const int L = p->L;
  const size_t bytes = sizeof(double2) * (size_t)B * L * L;
  cudaStream_t st = p->stream;
  p->launches = 0;
  double2* out = host ? p->d_out : (double2*)flm;
  bool halves = false;  // host buffers + blocked sweep: the batch is swept and copied out in two halves
  if (kind & OSPH_REAL) {
    if ((rc = forward_real(p, B, samples, flm, host))) return rc;
  } else if (p->windowed) {
    // factors do not fit at once: ring DFTs, then factor + sweep window by window
    const double2* src = (const double2*)samples;
    if (host) {
      CUDA_TRY(cudaMemcpyAsync(p->d_in, samples, bytes, cudaMemcpyHostToDevice, st));
      src = p->d_in;
    }
    CUDA_TRY(cudaEventRecord(p->ev[4], st));
    CUDA_TRY(launch_ring_forward(p, B, src));
    CUDA_TRY(cudaEventRecord(p->ev[5], st));
    CUDA_TRY(cudaEventRecord(p->ev[6], st));
    CUDA_TRY(cudaEventRecord(p->ev[7], st));
    CUDA_TRY(cudaEventRecord(p->ev[8], st));
    CUDA_TRY(forward_windows(p, B, out));
    p->last_sweep_kind = OSPH_SWEEP_WINDOWED;
    CUDA_TRY(cudaEventRecord(p->ev[9], st));
    CUDA_TRY(cudaEventRecord(p->ev_sweep_done, st));
    p->have_sweep_ev = true;
    if (host) CUDA_TRY(cudaMemcpyAsync(flm, p->d_out, bytes, cudaMemcpyDeviceToHost, st));
  } else if (!host) {
    // The factorisation reads nothing this call or earlier calls produce, so it
    // only waits for the previous forward's sweep (the last reader of the factor
    // buffers) and runs on a side stream beside whatever precedes this call on
    // the plan stream (e.g. the inverse of the same batch) and the ring DFTs.
    // OSPH_FACTOR_INLINE=1 (diagnostics): the factorisation on the plan stream, so
    // every stage is timed alone
    static const bool inline_factor = getenv("OSPH_FACTOR_INLINE") && atoi(getenv("OSPH_FACTOR_INLINE"));
    cudaStream_t sf = inline_factor ? st : p->s_in;
    if (inline_factor) {
    } else if (p->have_sweep_ev) {
      CUDA_TRY(cudaStreamWaitEvent(p->s_in, p->ev_sweep_done, 0));
    } else {
      CUDA_TRY(cudaEventRecord(p->ev_start, st));
      CUDA_TRY(cudaStreamWaitEvent(p->s_in, p->ev_start, 0));
    }
    CUDA_TRY(cudaEventRecord(p->ev[6], sf));
    CUDA_TRY(launch_factor(p, sf));
    CUDA_TRY(cudaEventRecord(p->ev[7], sf));
    CUDA_TRY(cudaEventRecord(p->ev[4], st));
    CUDA_TRY(launch_ring_forward(p, B, (const double2*)samples));
    CUDA_TRY(cudaEventRecord(p->ev[5], st));
    if (!inline_factor) CUDA_TRY(wait_factor_for_sweep(p, st));
  } else {
    // the factorisation needs no data: it runs while the samples are copied in,
    // and each chunk's ring DFTs start as soon as the chunk has landed
    const int nch = std::min(B, osph_plan::kIoChunks);
    CUDA_TRY(cudaEventRecord(p->ev_start, st));
    CUDA_TRY(cudaStreamWaitEvent(p->s_in, p->ev_start, 0));
    CUDA_TRY(cudaStreamWaitEvent(p->s_out, p->ev_start, 0));
    for (int c = 0; c < nch; ++c) {
      const int b0 = (int)((int64_t)B * c / nch), b1 = (int)((int64_t)B * (c + 1) / nch);
      const size_t off = (size_t)b0 * L * L, cb = sizeof(double2) * (size_t)(b1 - b0) * L * L;
      CUDA_TRY(cudaMemcpyAsync(p->d_in + off, (const double2*)samples + off, cb, cudaMemcpyHostToDevice, p->s_in));
      CUDA_TRY(cudaEventRecord(p->ev_in[c], p->s_in));
    }
    CUDA_TRY(cudaEventRecord(p->ev[6], st));
    CUDA_TRY(launch_factor(p, st));
    CUDA_TRY(cudaEventRecord(p->ev[7], st));
    // Blocked sweep, batches: two halves.  The first half's ring DFTs and sweep run while the
    // second half is still being copied in, and its coefficients go back to the host while the
    // second half is swept (PCIe is full duplex): the copies, not the kernels, bound this path.
    sweep_maps_per_team(p, B);  // decides the sweep (and the layout of the spectra)
    halves = p->sweep_blocked && nch == osph_plan::kIoChunks && B >= 16 && !ensure_sweep_blocked(p);
    for (int c = 0; c < nch; ++c) {
      const int b0 = (int)((int64_t)B * c / nch), b1 = (int)((int64_t)B * (c + 1) / nch);
      CUDA_TRY(cudaStreamWaitEvent(st, p->ev_in[c], 0));
      if (c == 0) CUDA_TRY(cudaEventRecord(p->ev[4], st));
      CUDA_TRY(launch_ring_forward(p, B, p->d_in, b0, b1 - b0));
      if (halves && (c == nch / 2 - 1 || c == nch - 1)) {
        const int h = c == nch - 1;
        const int hb0 = h ? (int)((int64_t)B * (nch / 2) / nch) : 0, hb1 = h ? B : (int)((int64_t)B * (nch / 2) / nch);
        const size_t off = (size_t)hb0 * L * L, hbytes = sizeof(double2) * (size_t)(hb1 - hb0) * L * L;
        if (h == 0) CUDA_TRY(cudaEventRecord(p->ev[8], st));
        const int nl = p->launches;
        CUDA_TRY(launch_sweep_blocked(p, hb1 - hb0, p->d_out + off, hb0));
        (void)nl;
        CUDA_TRY(cudaEventRecord(p->ev_done[h], st));
        CUDA_TRY(cudaStreamWaitEvent(p->s_out, p->ev_done[h], 0));
        CUDA_TRY(cudaMemcpyAsync((double2*)flm + off, p->d_out + off, hbytes, cudaMemcpyDeviceToHost, p->s_out));
      }
    }
    CUDA_TRY(cudaEventRecord(p->ev[5], st));
    if (halves) {
      p->last_sweep_kind = OSPH_SWEEP_BLOCKED;
      CUDA_TRY(cudaEventRecord(p->ev[9], st));
      CUDA_TRY(cudaEventRecord(p->ev_sweep_done, st));
      p->have_sweep_ev = true;
      CUDA_TRY(cudaEventRecord(p->ev_out, p->s_out));
      CUDA_TRY(cudaStreamWaitEvent(st, p->ev_out, 0));  // the plan stream covers the whole call
    }
  }
  if (!(kind & OSPH_REAL) && !p->windowed && !halves) {
    CUDA_TRY(cudaEventRecord(p->ev[8], st));
    CUDA_TRY(launch_sweep(p, B, out));
    p->last_sweep_kind = sweep_kind(p);
    CUDA_TRY(cudaEventRecord(p->ev[9], st));
    CUDA_TRY(cudaEventRecord(p->ev_sweep_done, st));
    p->have_sweep_ev = true;
    if (host) CUDA_TRY(cudaMemcpyAsync(flm, p->d_out, bytes, cudaMemcpyDeviceToHost, st));
  }
  p->have_fwd = true;
  if (kind & OSPH_ASYNC) return OSPH_OK;
  CUDA_TRY(cudaStreamSynchronize(st));
  if (stats) {
    float t01 = 0, t12 = 0, t23 = 0;
    cudaEventElapsedTime(&t01, p->ev[4], p->ev[5]);
    cudaEventElapsedTime(&t12, p->ev[6], p->ev[7]);
    cudaEventElapsedTime(&t23, p->ev[8], p->ev[9]);
    if (p->windowed) {
      window_times(p);
      t12 = p->last_factor_ms;
      t23 = p->last_sweep_ms;
    }
    stats->factor_seconds = t12 * 1e-3;
    stats->sweep_seconds = t23 * 1e-3;
    stats->solve_seconds = (t12 + t23) * 1e-3;
    stats->total_seconds = (t01 + t12 + t23) * 1e-3;
    stats->orders = L;
    stats->failed_order = -1;
    stats->failed_kappa = 0.0;
  }
  return forward_check(p, check, stats);
}

// check=True after a finished forward: the first failing order of the sweep
// (descending m, like the reference's loop) among the orders this plan factored.
int forward_check(osph_plan* p, int check, osph_stats* stats) {
  if (!check) return OSPH_OK;
  const int L = p->L;
  int lo, hi;
  own_orders(p, lo, hi);
  if (p->shard_mode == OSPH_SHARD_FACTORS) {  // the factors of every order were gathered
    lo = 0;
    hi = L - 1;
  }
  std::vector<double> kappa(L);
  std::vector<int> status(L);
  CUDA_TRY(cudaMemcpy(kappa.data(), p->d_kappa, sizeof(double) * L, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(status.data(), p->d_status, sizeof(int) * L, cudaMemcpyDeviceToHost));
  for (int m = hi; m >= lo; --m) {  // the reference raises at the first failing order of its sweep
    if (status[m] || !(kappa[m] <= 2.0e14)) {
      if (stats) {
        stats->failed_order = m;
        stats->failed_kappa = status[m] ? INFINITY : kappa[m];
      }
      char buf[160];
      snprintf(buf, sizeof buf, "order %d system is numerically singular (condition number %.3e)", m,
               status[m] ? INFINITY : kappa[m]);
      osph_set_error(buf);
      return OSPH_ERR_ILLCOND;
    }
  }
  return OSPH_OK;
}

extern "C" int osph_legendre_block(osph_plan* p, int m, double* out, int64_t ld, int kind) {
  DeviceGuard guard;
  g_last_error.clear();
  if (!p || !out) {
    osph_set_error("NULL plan or output pointer");
    return OSPH_ERR_ARG;
  }
  if (m < 0 || m >= p->L) {
    osph_set_error("order " + std::to_string(m) + " invalid for band limit " + std::to_string(p->L));
    return OSPH_ERR_ARG;
  }
  if (ld < p->L || !(kind & OSPH_DEVICE) || (kind & ~(OSPH_DEVICE | OSPH_ASYNC))) {
    osph_set_error("osph_legendre_block needs a device pointer and ld >= L");
    return OSPH_ERR_ARG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(launch_legendre_block(p, m, out, ld));
  if (!(kind & OSPH_ASYNC)) CUDA_TRY(cudaStreamSynchronize(p->stream));
  return OSPH_OK;
}

extern "C" int osph_ring_analysis(const double* ring, int n, int m, double* out, int device) {
  DeviceGuard guard;
  g_last_error.clear();
  if (!ring || !out) {
    osph_set_error("NULL pointer");
    return OSPH_ERR_ARG;
  }
  if (n < 1 || n % 2 == 0) {
    osph_set_error("ring length must be odd, got " + std::to_string(n));
    return OSPH_ERR_ARG;
  }
  const int k = (n - 1) / 2;
  if (m > k || -m > k) {
    osph_set_error("frequency " + std::to_string(m) + " is not resolvable on a ring of index " + std::to_string(k));
    return OSPH_ERR_ARG;
  }
  CUDA_TRY(cudaSetDevice(device));
  double2* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(double2) * (n + 2)));
  cudaError_t e = cudaMemcpy(d, ring, sizeof(double2) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_ring_pair(n, m, d, d + n, 0);
  if (e == cudaSuccess) e = cudaMemcpy(out, d + n, sizeof(double2) * 2, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) {
    osph_set_error(std::string("ring analysis: ") + cudaGetErrorString(e));
    return OSPH_ERR_CUDA;
  }
  return OSPH_OK;
}

extern "C" int osph_last_stage_times(const osph_plan* p, double* seconds) {
  DeviceGuard guard;
  if (!p || !seconds) {
    osph_set_error("NULL argument");
    return OSPH_ERR_ARG;
  }
  static const int pairs[6][2] = {{0, 1}, {1, 2}, {2, 3}, {4, 5}, {6, 7}, {8, 9}};
  for (int i = 0; i < 6; ++i) {
    float ms = 0.f;
    if (i < 3 ? p->have_inv : p->have_fwd) {
      CUDA_TRY(cudaEventSynchronize(p->ev[pairs[i][1]]));
      CUDA_TRY(cudaEventElapsedTime(&ms, p->ev[pairs[i][0]], p->ev[pairs[i][1]]));
      if (i >= 4 && p->windowed) {
        window_times(const_cast<osph_plan*>(p));
        ms = i == 4 ? p->last_factor_ms : p->last_sweep_ms;
      }
    }
    seconds[i] = ms * 1e-3;
  }
  return OSPH_OK;
}

extern "C" int osph_last_sweep_kind(const osph_plan* p) { return p ? p->last_sweep_kind : -1; }

extern "C" int osph_plan_pivots(osph_plan* p, int32_t* perm, double* seconds) {
  DeviceGuard guard;
  g_last_error.clear();
  if (!p) {
    osph_set_error("plan is NULL");
    return OSPH_ERR_ARG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  int rc;
  if ((rc = ensure_forward(p))) return rc;
  if (!p->piv_ready && (rc = discover_pivots(p))) return rc;
  if (perm) {
    const size_t npk = (size_t)p->L * (p->L + 1) / 2;
    CUDA_TRY(cudaMemcpy(perm, p->d_piv, sizeof(int32_t) * npk, cudaMemcpyDeviceToHost));
  }
  if (seconds) *seconds = p->pivot_seconds;
  return OSPH_OK;
}
