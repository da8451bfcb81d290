// shard.cu -- the transforms across several GPUs.
//
// The reference runs one process on one core (transform.py:347-467); its
// loops are what is partitioned here:
//   * the inverse's per-ring synthesis (transform.py:148-201, 334-344) is
//     independent per ring: a chain shard synthesises only its ring range;
//   * the forward's per-order factorisations (the solves of
//     transform.py:451) are independent per order: each shard factors a
//     block of orders, cost-balanced by sum (L-m)^3;
//   * the forward's order loop m = L-1 .. 0 (transform.py:441-463) is a
//     chain: order m reads the ring spectra after the corrections of every
//     order > m.  Blocks of orders descend with the rank, so a map's sweep
//     runs block after block: rank r sweeps its orders on the spectra it
//     received from rank r-1 (corrected by every higher order) and hands the
//     spectra and the coefficients solved so far to rank r+1.
// Batches instead split their maps over the GPUs; the factorisation is then
// split by order blocks and the factors all-gathered, so no GPU repeats the
// L^4/6 work of another.
//
// Two ways in:
//   * one process per GPU (torch.distributed over NCCL, or MPI): a plan is
//     made rank r of n by osph_plan_shard, the forward runs in stages
//     (osph_forward_stage) and the host moves the buffers osph_shard_buffer
//     points at (paper_1403_4661_b200/distributed.py);
//   * one process for all devices: osph_plan_create with ndev > 1 builds one
//     sub-plan per device and runs the same stages itself, moving the
//     buffers with peer-to-peer copies (cudaMemcpyPeerAsync over NVLink).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/osph.h"
#include "plan.cuh"

#define SH_TRY(expr)                                                          \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      osph_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));     \
      return OSPH_ERR_CUDA;                                                   \
    }                                                                         \
  } while (0)
#define SH_PEER_TRY(expr)                                                     \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      osph_set_error(std::string("peer exchange: ") + #expr + ": " + cudaGetErrorString(_e)); \
      return OSPH_ERR_NCCL;                                                   \
    }                                                                         \
  } while (0)

// ---------------------------------------------------------------------------
// partitions

// Blocks of orders, descending in m with the rank (rank 0 owns the highest
// orders), balanced by the factorisation cost sum (L - m)^3 (2 n^3 flops per
// order); every rank owns at least one order.
static void order_blocks(int L, int n, std::vector<int>& lo, std::vector<int>& hi) {
  lo.assign(n, 0);
  hi.assign(n, -1);
  double total = 0.0;
  for (int m = 0; m < L; ++m) total += std::pow((double)(L - m), 3.0);
  std::vector<int> owner(L);
  double acc = 0.0;
  for (int m = L - 1; m >= 0; --m) {
    const double c = std::pow((double)(L - m), 3.0);
    owner[m] = std::min(n - 1, (int)((double)n * (acc + 0.5 * c) / total));
    acc += c;
  }
  // the cubic weights can leave a rank empty at small L: fall back to equal counts
  std::vector<int> cnt(n, 0);
  for (int m = 0; m < L; ++m) cnt[owner[m]]++;
  if (std::any_of(cnt.begin(), cnt.end(), [](int c) { return c == 0; }))
    for (int m = 0; m < L; ++m) owner[m] = (int)((int64_t)(L - 1 - m) * n / L);
  for (int r = 0; r < n; ++r) {
    lo[r] = L;
    hi[r] = -1;
  }
  for (int m = 0; m < L; ++m) {
    lo[owner[m]] = std::min(lo[owner[m]], m);
    hi[owner[m]] = std::max(hi[owner[m]], m);
  }
}

extern "C" int osph_shard_range(int L, int rank, int nranks, int mode, int* m_lo, int* m_hi, int* k_lo, int* k_hi) {
  if (L < 1 || nranks < 1 || nranks > L || rank < 0 || rank >= nranks ||
      (mode != OSPH_SHARD_CHAIN && mode != OSPH_SHARD_FACTORS)) {
    osph_set_error("osph_shard_range: need 0 <= rank < nranks <= L and a shard mode");
    return OSPH_ERR_ARG;
  }
  std::vector<int> lo, hi;
  order_blocks(L, nranks, lo, hi);
  if (m_lo) *m_lo = lo[rank];
  if (m_hi) *m_hi = hi[rank];
  const bool chain = mode == OSPH_SHARD_CHAIN;
  if (k_lo) *k_lo = chain ? (int)((int64_t)L * rank / nranks) : 0;
  if (k_hi) *k_hi = chain ? (int)((int64_t)L * (rank + 1) / nranks) : L;
  return OSPH_OK;
}

extern "C" int osph_plan_shard(osph_plan* p, int rank, int nranks, int mode) {
  DeviceGuard guard;
  if (!p || !p->group.empty() || !p->group_maps.empty() || !p->group_devs.empty()) {
    osph_set_error("osph_plan_shard needs a single-device plan");
    return OSPH_ERR_ARG;
  }
  if (p->fwd_ready || p->shard_mode) {
    osph_set_error("osph_plan_shard must come before the plan's first forward (and only once)");
    return OSPH_ERR_ARG;
  }
  int mlo, mhi, klo, khi, rc;
  if ((rc = osph_shard_range(p->L, rank, nranks, mode, &mlo, &mhi, &klo, &khi))) return rc;
  SH_TRY(cudaSetDevice(p->device));
  p->shard_mode = mode;
  p->shard_rank = rank;
  p->shard_n = nranks;
  p->own_m_lo = mlo;
  p->own_m_hi = mhi;
  p->sweep_cfg_B = -1;
  if (mode != OSPH_SHARD_CHAIN) return OSPH_OK;
  // the inverse of a chain shard: rings [klo, khi) only
  p->own_k_lo = klo;
  p->own_k_hi = khi;
  std::vector<int> ord, blu;
  for (int k : p->h_ring_order)
    if (k >= klo && k < khi) ord.push_back(k);
  int nbig = 0, nreg = 0, nreg2 = 0;
  for (int k : p->h_bluestein_rings)  // largest first: the 16384-point rings lead, the register-resident ones trail
    if (k >= klo && k < khi) {
      blu.push_back(k);
      if (p->h_fft_n[k] > OSPH_FFT_MAX) ++nbig;
      if (p->h_fft_n[k] <= p->reg_fft_max) ++nreg;
      if (p->h_fft_n[k] <= p->reg_fft_max && p->h_fft_n[k] == 2048) ++nreg2;
    }
  int* d_ord = nullptr;
  int* d_blu = nullptr;
  SH_TRY(cudaMalloc(&d_ord, sizeof(int) * std::max<size_t>(1, ord.size())));
  SH_TRY(cudaMalloc(&d_blu, sizeof(int) * std::max<size_t>(1, blu.size())));
  if (!ord.empty()) SH_TRY(cudaMemcpy(d_ord, ord.data(), sizeof(int) * ord.size(), cudaMemcpyHostToDevice));
  if (!blu.empty()) SH_TRY(cudaMemcpy(d_blu, blu.data(), sizeof(int) * blu.size(), cudaMemcpyHostToDevice));
  p->d_inv_ring_order = d_ord;
  p->inv_nr = (int)ord.size();
  p->d_inv_bluestein = d_blu;
  p->inv_n_bluestein = p->dft_ok ? (int)blu.size() : 0;
  p->inv_n_big = p->dft_ok ? nbig : 0;
  p->inv_n_reg = p->dft_ok ? nreg : 0;
  p->inv_n_reg2 = p->dft_ok ? nreg2 : 0;
  p->inv_direct_lo = std::min(klo, p->n_direct_rings);
  p->inv_direct_hi = std::min(khi, p->n_direct_rings);
  p->inv_own_lists = true;
  return OSPH_OK;
}

// ---------------------------------------------------------------------------
// exchange buffers

static int buffer_span(osph_plan* p, int which, int B, int m_lo, int m_hi, void** ptr, int64_t* bytes) {
  const int L = p->L;
  *ptr = nullptr;
  *bytes = 0;
  if (which == OSPH_BUF_SPECTRA) {
    if (B < 1 || B > p->max_batch) {
      osph_set_error("spectra: batch outside [1, max_batch]");
      return OSPH_ERR_ARG;
    }
    if (!p->windowed && !p->sweep_large) {
      osph_set_error("spectra are exchanged only by chain-sharded (windowed) plans");
      return OSPH_ERR_ARG;
    }
    *ptr = p->d_r;
    *bytes = (int64_t)sizeof(double2) * L * (L + 1) * B;  // [B][pos][+-], plain layout
    return OSPH_OK;
  }
  if (m_lo < 0 || m_hi >= L || m_lo > m_hi) {
    osph_set_error("order range outside [0, L)");
    return OSPH_ERR_ARG;
  }
  if (p->windowed) {
    osph_set_error("factor buffers are exchanged only by resident (factor-sharded) plans");
    return OSPH_ERR_ARG;
  }
  const int cnt = m_hi - m_lo + 1;
  switch (which) {
    case OSPH_BUF_XT:
      *ptr = p->d_xt + p->h_xt_off[m_lo];
      *bytes = (int64_t)sizeof(double) * (p->h_xt_off[m_hi + 1] - p->h_xt_off[m_lo]);
      break;
    case OSPH_BUF_PB:
      *ptr = p->d_pbelow + p->h_pb_off[m_lo];
      *bytes = (int64_t)sizeof(double) * (p->h_pb_off[m_hi + 1] - p->h_pb_off[m_lo]);
      break;
    case OSPH_BUF_AT:
      if (p->d_at) {
        *ptr = p->d_at + p->h_xt_off[m_lo];
        *bytes = (int64_t)sizeof(double) * (p->h_xt_off[m_hi + 1] - p->h_xt_off[m_lo]);
      }
      break;
    case OSPH_BUF_U:
      *ptr = p->d_u + (int64_t)m_lo * uw_ld(L);
      *bytes = (int64_t)sizeof(double) * cnt * uw_ld(L);
      break;
    case OSPH_BUF_W:
      *ptr = p->d_w + (int64_t)m_lo * uw_ld(L);
      *bytes = (int64_t)sizeof(double) * cnt * uw_ld(L);
      break;
    case OSPH_BUF_BETA:
      *ptr = p->d_beta + m_lo;
      *bytes = (int64_t)sizeof(double) * cnt;
      break;
    case OSPH_BUF_JSTAR:
      *ptr = p->d_jstar + m_lo;
      *bytes = (int64_t)sizeof(int) * cnt;
      break;
    case OSPH_BUF_NORMS:
      *ptr = p->d_norms + 2 * (int64_t)m_lo;
      *bytes = (int64_t)sizeof(unsigned long long) * 2 * cnt;
      break;
    case OSPH_BUF_STATUS:
      *ptr = p->d_status + m_lo;
      *bytes = (int64_t)sizeof(int) * cnt;
      break;
    case OSPH_BUF_UT:
      if (p->d_ut) {
        *ptr = p->d_ut + p->h_ut_off[m_lo];
        *bytes = (int64_t)sizeof(double) * (p->h_ut_off[m_hi + 1] - p->h_ut_off[m_lo]);
      }
      break;
    default:
      osph_set_error("unknown buffer id");
      return OSPH_ERR_ARG;
  }
  return OSPH_OK;
}

extern "C" int osph_shard_buffer(osph_plan* p, int which, int B, int m_lo, int m_hi, void** ptr, int64_t* bytes) {
  DeviceGuard guard;
  if (!p || !ptr || !bytes || !p->group_devs.empty()) {
    osph_set_error("osph_shard_buffer: NULL argument or multi-device plan");
    return OSPH_ERR_ARG;
  }
  SH_TRY(cudaSetDevice(p->device));
  int rc;
  if ((rc = ensure_forward(p))) return rc;
  return buffer_span(p, which, B, m_lo, m_hi, ptr, bytes);
}

// ---------------------------------------------------------------------------
// staged forward

int forward_stage_enqueue(osph_plan* p, int stages, int B, const void* samples, void* flm) {
  int rc;
  SH_TRY(cudaSetDevice(p->device));
  if ((rc = ensure_forward(p))) return rc;
  if (!p->piv_ready && (rc = discover_pivots(p))) return rc;
  p->need_norms = true;
  cudaStream_t st = p->stream;
  if (stages & OSPH_STAGE_RINGS) {
    SH_TRY(cudaEventRecord(p->ev[4], st));
    SH_TRY(launch_ring_forward(p, B, (const double2*)samples));
    SH_TRY(cudaEventRecord(p->ev[5], st));
  }
  if (stages & OSPH_STAGE_FACTOR) {
    SH_TRY(cudaEventRecord(p->ev[6], st));
    if (p->windowed) SH_TRY(forward_windows_factor_first(p));
    else SH_TRY(launch_factor(p, st));
    SH_TRY(cudaEventRecord(p->ev[7], st));
  }
  if (stages & OSPH_STAGE_SWEEP) {
    SH_TRY(cudaEventRecord(p->ev[8], st));
    if (p->windowed) {
      SH_TRY(forward_windows_sweep(p, B, (double2*)flm));
      p->last_sweep_kind = OSPH_SWEEP_WINDOWED;
    } else {
      if (p->shard_mode == OSPH_SHARD_FACTORS) SH_TRY(launch_kappa(p, st));  // norms gathered from every shard
      SH_TRY(launch_sweep(p, B, (double2*)flm));
      p->last_sweep_kind = p->sweep_blocked ? OSPH_SWEEP_BLOCKED : p->sweep_gemm ? OSPH_SWEEP_GEMM : p->sweep_large ? OSPH_SWEEP_LARGE : OSPH_SWEEP_PERSISTENT;
    }
    SH_TRY(cudaEventRecord(p->ev[9], st));
    SH_TRY(cudaEventRecord(p->ev_sweep_done, st));
    p->have_sweep_ev = true;
  }
  p->have_fwd = true;
  return OSPH_OK;
}

extern "C" int osph_forward_stage(osph_plan* p, int stages, int B, const void* samples, void* flm, int kind,
                                  int check, osph_stats* stats) {
  DeviceGuard guard;
  if (!p || !p->group_devs.empty()) {
    osph_set_error("osph_forward_stage needs a single-device plan");
    return OSPH_ERR_ARG;
  }
  if (!(kind & OSPH_DEVICE) || (kind & OSPH_REAL) || (kind & ~(OSPH_DEVICE | OSPH_ASYNC))) {
    osph_set_error("osph_forward_stage takes device pointers of complex maps (OSPH_DEVICE [| OSPH_ASYNC])");
    return OSPH_ERR_ARG;
  }
  if (stages <= 0 || (stages & ~(OSPH_STAGE_RINGS | OSPH_STAGE_FACTOR | OSPH_STAGE_SWEEP))) {
    osph_set_error("unknown forward stages");
    return OSPH_ERR_ARG;
  }
  if (((stages & OSPH_STAGE_RINGS) && !samples) || ((stages & OSPH_STAGE_SWEEP) && !flm)) {
    osph_set_error("NULL data pointer");
    return OSPH_ERR_ARG;
  }
  if ((stages & (OSPH_STAGE_RINGS | OSPH_STAGE_SWEEP)) && (B < 1 || B > p->max_batch)) {
    osph_set_error("batch " + std::to_string(B) + " outside [1, max_batch=" + std::to_string(p->max_batch) + "]");
    return OSPH_ERR_ARG;
  }
  if ((kind & OSPH_ASYNC) && check) {
    osph_set_error("check=1 needs a host-blocking call");
    return OSPH_ERR_ARG;
  }
  int rc;
  if ((rc = forward_stage_enqueue(p, stages, B, samples, flm))) return rc;
  if (kind & OSPH_ASYNC) return OSPH_OK;
  SH_TRY(cudaStreamSynchronize(p->stream));
  if (stats) {
    *stats = osph_stats{};
    stats->orders = p->L;
    stats->failed_order = -1;
  }
  if ((stages & OSPH_STAGE_SWEEP) && check) return forward_check(p, check, stats);
  return OSPH_OK;
}

// ---------------------------------------------------------------------------
// one process, several devices (osph_plan_create with ndev > 1)

int group_create(int L, const double* thetas, int max_batch, int ndev, const int* devs, osph_plan** out) {
  if (!out || !thetas || L < 1 || L > 4096 || max_batch < 1) {
    osph_set_error("osph_plan_create: bad arguments");
    return OSPH_ERR_ARG;
  }
  if (ndev > L) {
    osph_set_error("more devices than orders");
    return OSPH_ERR_ARG;
  }
  int count = 0;
  SH_TRY(cudaGetDeviceCount(&count));
  for (int i = 0; i < ndev; ++i)
    if (devs[i] < 0 || devs[i] >= count) {
      osph_set_error("device ordinal out of range");
      return OSPH_ERR_ARG;
    }
  for (int k = 0; k < L; ++k)
    if (!(thetas[k] > 0.0 && thetas[k] <= OSPH_PI)) {
      osph_set_error("co-latitudes must lie in (0, pi]");
      return OSPH_ERR_ARG;
    }
  // NVLink peer access between every pair of distinct devices (P2P copies; best effort)
  for (int i = 0; i < ndev; ++i)
    for (int j = 0; j < ndev; ++j) {
      if (devs[i] == devs[j]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devs[i], devs[j]);
      if (can) {
        cudaSetDevice(devs[i]);
        cudaDeviceEnablePeerAccess(devs[j], 0);
        cudaGetLastError();  // already enabled is fine
      }
    }
  osph_plan* p = new osph_plan();
  p->L = L;
  p->max_batch = max_batch;
  p->device = devs[0];
  p->group_devs.assign(devs, devs + ndev);
  p->h_thetas.assign(thetas, thetas + L);
  p->dft_ok = true;
  *out = p;
  return OSPH_OK;
}

// Lazily build the per-device sub-plans of one kind.
static int group_subs(osph_plan* p, int mode) {
  std::vector<osph_plan*>& subs = mode == OSPH_SHARD_CHAIN ? p->group : p->group_maps;
  if (!subs.empty()) return OSPH_OK;
  const int n = (int)p->group_devs.size();
  const int mb = mode == OSPH_SHARD_CHAIN ? p->max_batch : (p->max_batch + n - 1) / n;
  for (int i = 0; i < n; ++i) {
    osph_plan* q = nullptr;
    int rc = plan_create_one(p->L, p->h_thetas.data(), std::max(1, mb), p->group_devs[i], &q);
    if (!rc) rc = osph_plan_shard(q, i, n, mode);
    if (rc) {
      plan_free(q);
      for (osph_plan* s : subs) plan_free(s);
      subs.clear();
      return rc;
    }
    subs.push_back(q);
  }
  return OSPH_OK;
}

static void split_maps(int B, int n, int i, int& b0, int& b1) {
  b0 = (int)((int64_t)B * i / n);
  b1 = (int)((int64_t)B * (i + 1) / n);
}

static int sync_all(const std::vector<osph_plan*>& subs) {
  for (osph_plan* q : subs) {
    SH_TRY(cudaSetDevice(q->device));
    SH_TRY(cudaStreamSynchronize(q->stream));
  }
  return OSPH_OK;
}

int group_inverse(osph_plan* p, int B, const void* flm, void* samples, int kind) {
  const int n = (int)p->group_devs.size();
  if (kind & ~(OSPH_REAL)) {
    osph_set_error("multi-device plans take host pointers (the plan owns every device's buffers)");
    return OSPH_ERR_ARG;
  }
  if (B < 1 || B > p->max_batch || !flm || !samples) {
    osph_set_error("batch outside [1, max_batch] or NULL data pointer");
    return OSPH_ERR_ARG;
  }
  const size_t per_map = (size_t)p->L * p->L;
  int rc;
  if (B >= n) {  // maps split over the devices
    if ((rc = group_subs(p, OSPH_SHARD_FACTORS))) return rc;
    for (int i = 0; i < n; ++i) {
      int b0, b1;
      split_maps(B, n, i, b0, b1);
      if ((rc = inverse_enqueue(p->group_maps[i], b1 - b0, (const double2*)flm + b0 * per_map,
                                (double2*)samples + b0 * per_map, kind)))
        return rc;
    }
    return sync_all(p->group_maps);
  }
  if (kind & OSPH_REAL) {
    osph_set_error("OSPH_REAL needs at least one map per device");
    return OSPH_ERR_ARG;
  }
  // one map chain: every device synthesises its ring range of every map
  if ((rc = group_subs(p, OSPH_SHARD_CHAIN))) return rc;
  for (int i = 0; i < n; ++i)
    if ((rc = inverse_enqueue(p->group[i], B, flm, samples, kind))) return rc;
  return sync_all(p->group);
}

int group_forward(osph_plan* p, int B, const void* samples, void* flm, int kind, int check, osph_stats* stats) {
  const int n = (int)p->group_devs.size();
  const int L = p->L;
  if (kind & ~(OSPH_REAL)) {
    osph_set_error("multi-device plans take host pointers (the plan owns every device's buffers)");
    return OSPH_ERR_ARG;
  }
  if (B < 1 || B > p->max_batch || !flm || !samples) {
    osph_set_error("batch outside [1, max_batch] or NULL data pointer");
    return OSPH_ERR_ARG;
  }
  if (kind & OSPH_REAL) {
    osph_set_error("multi-device forward: complex maps only");
    return OSPH_ERR_ARG;
  }
  const auto t0 = std::chrono::steady_clock::now();
  const size_t per_map = (size_t)L * L;
  int rc;
  if (B >= n) {
    // ---- batch: factor by order blocks, all-gather the factors peer to peer, sweep own maps
    if ((rc = group_subs(p, OSPH_SHARD_FACTORS))) return rc;
    std::vector<osph_plan*>& s = p->group_maps;
    for (int i = 0; i < n; ++i) {
      SH_TRY(cudaSetDevice(s[i]->device));
      if ((rc = ensure_io(s[i]))) return rc;
      if ((rc = forward_stage_enqueue(s[i], OSPH_STAGE_FACTOR, 0, nullptr, nullptr))) return rc;
      SH_TRY(cudaEventRecord(s[i]->ev_start, s[i]->stream));  // factors of block i complete
    }
    for (int d = 0; d < n; ++d) {
      SH_TRY(cudaSetDevice(s[d]->device));
      for (int q = 0; q < n; ++q) {
        if (q == d) continue;
        SH_TRY(cudaStreamWaitEvent(s[d]->stream, s[q]->ev_start, 0));
        for (int which = OSPH_BUF_XT; which < OSPH_BUF_COUNT; ++which) {
          void *src, *dst;
          int64_t bs, bd;
          if ((rc = buffer_span(s[q], which, 1, s[q]->own_m_lo, s[q]->own_m_hi, &src, &bs))) return rc;
          if ((rc = buffer_span(s[d], which, 1, s[q]->own_m_lo, s[q]->own_m_hi, &dst, &bd))) return rc;
          if (bs > 0) SH_PEER_TRY(cudaMemcpyPeerAsync(dst, s[d]->device, src, s[q]->device, (size_t)bs, s[d]->stream));
        }
      }
    }
    for (int i = 0; i < n; ++i) {
      int b0, b1;
      split_maps(B, n, i, b0, b1);
      const int bi = b1 - b0;
      SH_TRY(cudaSetDevice(s[i]->device));
      SH_TRY(cudaMemcpyAsync(s[i]->d_in, (const double2*)samples + b0 * per_map, sizeof(double2) * bi * per_map,
                             cudaMemcpyHostToDevice, s[i]->stream));
      if ((rc = forward_stage_enqueue(s[i], OSPH_STAGE_RINGS | OSPH_STAGE_SWEEP, bi, s[i]->d_in, s[i]->d_out)))
        return rc;
      SH_TRY(cudaMemcpyAsync((double2*)flm + b0 * per_map, s[i]->d_out, sizeof(double2) * bi * per_map,
                             cudaMemcpyDeviceToHost, s[i]->stream));
    }
    // every device's gathered factors are read by its own sweep only; the owners' next
    // factorisation (next call) starts after this call returns
    if ((rc = sync_all(s))) return rc;
    if (stats) {
      *stats = osph_stats{};
      stats->orders = L;
      stats->failed_order = -1;
    }
    for (int i = 0; i < n && check; ++i)
      if ((rc = forward_check(s[i], check, stats))) return rc;
  } else {
    // ---- one map chain: blocks of orders, spectra + coefficients handed down the chain
    if ((rc = group_subs(p, OSPH_SHARD_CHAIN))) return rc;
    std::vector<osph_plan*>& s = p->group;
    for (int i = 0; i < n; ++i) {
      SH_TRY(cudaSetDevice(s[i]->device));
      if ((rc = ensure_io(s[i]))) return rc;
      if ((rc = ensure_forward(s[i]))) return rc;
    }
    // rank 0 transforms the rings (the spectra travel with the chain); every rank factors its block
    SH_TRY(cudaSetDevice(s[0]->device));
    SH_TRY(cudaMemcpyAsync(s[0]->d_in, samples, sizeof(double2) * B * per_map, cudaMemcpyHostToDevice, s[0]->stream));
    if ((rc = forward_stage_enqueue(s[0], OSPH_STAGE_RINGS | OSPH_STAGE_FACTOR, B, s[0]->d_in, s[0]->d_out)))
      return rc;
    for (int i = 1; i < n; ++i) {
      SH_TRY(cudaSetDevice(s[i]->device));
      if ((rc = forward_stage_enqueue(s[i], OSPH_STAGE_FACTOR, B, nullptr, nullptr))) return rc;
      SH_TRY(cudaEventRecord(s[i]->ev_start, s[i]->stream));
    }
    for (int r = 0; r < n; ++r) {
      SH_TRY(cudaSetDevice(s[r]->device));
      if ((rc = forward_stage_enqueue(s[r], OSPH_STAGE_SWEEP, B, nullptr, s[r]->d_out))) return rc;
      if (r + 1 < n) {
        // hand-off: spectra (corrected by every order >= this block) and coefficients so far;
        // the receiver's own stream waits for its factorisation (ev_start) before the copies land
        osph_plan* nx = s[r + 1];
        void *src, *dst;
        int64_t bytes, b2;
        if ((rc = buffer_span(s[r], OSPH_BUF_SPECTRA, B, 0, 0, &src, &bytes))) return rc;
        if ((rc = buffer_span(nx, OSPH_BUF_SPECTRA, B, 0, 0, &dst, &b2))) return rc;
        SH_TRY(cudaEventRecord(s[r]->ev_out, s[r]->stream));
        SH_TRY(cudaSetDevice(nx->device));
        SH_TRY(cudaStreamWaitEvent(nx->stream, s[r]->ev_out, 0));
        SH_PEER_TRY(cudaMemcpyPeerAsync(dst, nx->device, src, s[r]->device, (size_t)bytes, nx->stream));
        SH_PEER_TRY(cudaMemcpyPeerAsync(nx->d_out, nx->device, s[r]->d_out, s[r]->device,
                                        sizeof(double2) * B * per_map, nx->stream));
      }
    }
    osph_plan* last = s[n - 1];
    SH_TRY(cudaSetDevice(last->device));
    SH_TRY(cudaMemcpyAsync(flm, last->d_out, sizeof(double2) * B * per_map, cudaMemcpyDeviceToHost, last->stream));
    if ((rc = sync_all(s))) return rc;
    if (stats) {
      *stats = osph_stats{};
      stats->orders = L;
      stats->failed_order = -1;
    }
    for (int r = 0; r < n && check; ++r)  // highest failing order first: rank 0 holds the top block
      if ((rc = forward_check(s[r], check, stats))) return rc;
  }
  if (stats) {
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    stats->total_seconds = sec;
    stats->solve_seconds = sec;
  }
  return OSPH_OK;
}
