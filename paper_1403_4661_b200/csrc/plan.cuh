// plan.cuh -- internal plan object and kernel launchers of libosph.
#pragma once
#include <string>
#include <vector>

#include "common.cuh"
#include "../../include/osph.h"

struct BfStep {
  int cnt = 0, pre_panel = 0, n_panel = 0, pre_upd = 0, n_upd = 0, pre_updw = 0, n_updw = 0;  // updw: 128-row tiles
};
struct BfPairStep {  // one paired (rank-128) step of factor_bf.cu: panels J1 = [j0, j0+64), J2 = [j0+64, j0+128)
  int j0 = 0, cnt = 0, cnt2 = 0;  // orders with n > j0 / with n > j0 + 64 (the first ones of the range)
  int pre_panel = 0, n_panel = 0, n_panel2 = 0;  // 64-row tiles per order (n_panel2: first cnt2 orders)
  int pre_row = 0, n_row = 0;                    // column tiles outside J1, J2 (cnt2 orders)
  int pre_upd2 = 0, n_upd2 = 0, pre_updw2 = 0, n_updw2 = 0;        // paired update, 64- / 128-row tiles
  int pre_single = 0, n_single = 0, pre_singlew = 0, n_singlew = 0;  // orders cnt2..cnt-1: rank-64 update
};
struct BfRange {  // work-item tables of one range of orders (factor_bf.cu)
  int m_first = -1, m_last = -1;
  std::vector<BfStep> steps;
  std::vector<BfPairStep> psteps;
  int* d_tab = nullptr;
  double* dbuf = nullptr;  // this range's diagonal-block inverses (nullptr: the plan's d_bf_d)
};
struct BfOffsets {  // per-order offsets (indexed by m) into the factor buffers
  const int64_t* ainv;
  const int64_t* xt;
  const int64_t* pb;
  const int64_t* bf;
};
struct FwdWindow {  // orders m_lo..m_hi, factored then swept together
  int m_lo = 0, m_hi = 0;
  BfRange bf;
  int64_t* d_offs = nullptr;  // 4 x (L+1): ainv, xt, pb, bf offsets (window-relative)
  cudaEvent_t ev[4] = {};     // factor start/end, sweep start/end
};

struct SpinState {  // spin-weighted transforms of one spin s != 0 (spin.cu); u = signed order + L - 1
  int s = 0;
  int* d_ls = nullptr;          // [2L-1][L] first degree whose value is in the double range (L: none)
  double2* d_pstart = nullptr;  // [2L-1][L] {sY_(ls-1), sY_ls} (true values)
  double4* d_rec = nullptr;     // [2L-1][L] {alpha, beta, gamma, 0}: sY_(l+1) = (alpha x - beta) sY_l - gamma sY_(l-1)
  double* d_x = nullptr;        // X_u = least-squares solution operator, row-major (L - lo) x (L - m)
  std::vector<int64_t> h_x_off;  // [2L] offsets into d_x
  int64_t* d_x_off = nullptr;
  double* d_pb = nullptr;        // Pb_u = 2pi sY_l(u)(theta_k), rings k < m, row-major m x (L - lo)
  std::vector<int64_t> h_pb_off;  // [2L]
  int64_t* d_pb_off = nullptr;
  double* d_kappa = nullptr;     // [2L-1] ||A_u||_1 ||X_u||_1 (infinity: singular / non-finite)
  std::vector<double> h_kappa;
  bool factored = false;
  double factor_seconds = 0.0;   // device time of the last factorisation (0 once cached)
};

struct osph_plan {
  int L = 0;
  int device = 0;
  int max_batch = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int launches = 0;  // kernels enqueued by the last transform call

  // ---- grid + recurrence tables (O(L^2), built once per plan) ----
  double* d_cos = nullptr;  // [L] cos(theta_k)
  double* d_sin = nullptr;  // [L] sin(theta_k)
  double2* d_rec = nullptr;   // packed (m, l): {a_lm, 1/a_(l+1)m}
  int* d_ls = nullptr;        // [m][k] first degree whose value is in the double range
  double2* d_pstart = nullptr;  // [m][k] {P_(ls-1)m, P_(ls)m} (true values)
  int* d_ring_order = nullptr;  // [L] rings sorted by sin(theta), for warp-coherent skipping
  std::vector<int> h_ring_order, h_bluestein_rings;  // host copies (shard ring lists are filtered from them)

  // ---- ring DFT tables ----
  std::vector<int> h_fft_n;          // [L] Bluestein FFT size per ring (0 = direct DFT)
  std::vector<int64_t> h_chirp_off;  // [L] offset of chirp table (n entries)
  std::vector<int64_t> h_bhat_off;   // [L] offset of FFT(kernel) tables (2N entries: fwd, inv)
  int* d_fft_n = nullptr;
  int64_t* d_chirp_off = nullptr;
  int64_t* d_bhat_off = nullptr;
  double2* d_chirp = nullptr;  // e^{i pi t^2 / n}
  double2* d_bhat = nullptr;   // FFT_N of the conjugate chirp kernel (per direction, / N)
  double2* d_tw = nullptr;     // e^{-2 pi i j / OSPH_FFT_MAX}, j < OSPH_FFT_MAX/2
  double2* d_roots = nullptr;  // small rings: e^{2 pi i r / n} at k*k + r (k*k < direct limit)
  int n_bluestein_rings = 0;
  int* d_bluestein_rings = nullptr;  // ring ids that use Bluestein, largest first
  int n_direct_rings = 0;
  int n_big_rings = 0;  // rings with a 16384-point Bluestein FFT (2-CTA clusters; first in d_bluestein_rings)
  double2* d_sw = nullptr;  // [OSPH_SW_GLOBAL] per-stage FFT twiddles (fft.cuh)
  double2* d_rtw = nullptr;  // [OSPH_RTW_SIZE] inter-pass twiddles of the register-resident FFTs (fft_reg.cuh)
  int reg_fft_max = 0;       // rings with fft_n <= this run the register-resident kernels (kernel spectra in natural order)
  int n_reg_rings = 0;       // how many: the LAST n_reg_rings entries of d_bluestein_rings (sorted largest first)
  int inv_n_reg = 0;         // the same count for d_inv_bluestein
  int n_reg2_rings = 0, inv_n_reg2 = 0;  // of those, the 2048-point rings (they lead the register-resident ones)
  bool dft_ok = true;  // every ring's Bluestein FFT fits one CTA (else: tables-only plan)
  // rings the INVERSE produces: all of them, or a chain shard's contiguous range
  // [own_k_lo, own_k_hi) (osph_plan_shard); the forward ring DFTs always cover all rings
  int inv_nr = 0;                   // rings in d_inv_ring_order (synthesis ring list)
  int* d_inv_ring_order = nullptr;  // those rings sorted by sin(theta) (aliases d_ring_order when unsharded)
  int* d_inv_bluestein = nullptr;   // their Bluestein rings, 16384-point ones first (aliases d_bluestein_rings)
  int inv_n_bluestein = 0, inv_n_big = 0, inv_direct_lo = 0, inv_direct_hi = 0;
  bool inv_own_lists = false;       // d_inv_* are separate allocations (free them)

  // ---- sharding over GPUs (osph_plan_shard) ----
  int shard_mode = 0;               // 0 none, OSPH_SHARD_CHAIN, OSPH_SHARD_FACTORS
  int shard_rank = 0, shard_n = 1;
  int own_m_lo = 0, own_m_hi = -1;  // orders this plan factors (and, in chain mode, sweeps); -1: all
  int own_k_lo = 0, own_k_hi = 0;   // rings this plan synthesises in the inverse
  // multi-device plan (osph_plan_create with ndev > 1): per-device sub-plans, created lazily:
  // chain shards (B < ndev: one map across the devices) and factor shards (B >= ndev: maps split)
  std::vector<int> group_devs;
  std::vector<osph_plan*> group, group_maps;
  std::vector<double> h_thetas;

  // ---- forward factor storage (per call, data independent) ----
  std::vector<int64_t> h_ainv_off;  // [L+1] offset of order m's n x n inverse
  std::vector<int64_t> h_pb_off;    // [L+1] offset of order m's (m x n) below-block
  int64_t* d_ainv_off = nullptr;
  int64_t* d_pb_off = nullptr;
  double* d_ainv = nullptr;
  double* d_pbelow = nullptr;
  int* d_piv = nullptr;          // [pos(m, j)] row permutation of order m's inverse
  unsigned long long* d_norms = nullptr;  // [2L] ||A_m||_1, ||A_m^-1||_1 (as ordered bits)
  double* d_kappa = nullptr;     // [L] 1-norm condition estimate per order
  int* d_status = nullptr;       // [L] 0 ok, 1 zero/non-finite pivot
  int* d_jstar = nullptr;        // [L] column of X_m fed by ring m (perm[j*] = 0)
  double* d_beta = nullptr;      // [L] beta_m = Pb_m[m-1, :] . X_m[:, j*]
  double* d_u = nullptr;         // [L][L] u_m = Pb_m[m-1, :] X_m P^T (chain partial a_{m-1} = u_m . rhs_m)
  double* d_w = nullptr;         // [L][L] w_m = X_m[:, j*] (late-entry column)
  std::vector<int64_t> h_xt_off;  // [L+1] offset of order m's 8-row-tiled inverse
  int64_t* d_xt_off = nullptr;
  double* d_xt = nullptr;         // X_m in 8-row tiles (sweep operand)
  // blocked sweep (sweep_block.cu): coupling rows U_m (tiled), per-block scratch
  std::vector<int64_t> h_ut_off;  // [L+1]
  int64_t* d_ut_off = nullptr;
  double* d_ut = nullptr;
  double2* d_sb_x = nullptr;      // [block][B][+-][L] solved coefficients of a block of orders
  double2* d_sb_a = nullptr;      // [block][32][B][+-] coupling products U_s g_s
  double2* d_sb_g = nullptr;      // [block][16][B][+-] corrections of a block through the short rings k < 16
  double2* d_sb_r2 = nullptr;     // opposite-tone corrections, laid out like R (zero between forward calls)
  bool sweep_blocked = false;     // batches: orders peeled in blocks, three batched GEMM launches per block
  bool fwd_ready = false;        // forward buffers allocated
  bool piv_ready = false;        // d_piv holds the (grid-determined) pivot order of every order
  double pivot_seconds = 0.0;    // host wall time of this plan's pivot discovery (0: cached per grid)
  int last_sweep_kind = -1;      // OSPH_SWEEP_* of the last forward call
  int sweep_cfg_B = -1;          // cached sweep launch configuration for batch sweep_cfg_B
  int sweep_cfg[3] = {0, 0, 0};  // maps per team, cluster width, ring stages
  bool sweep_large = false;      // L > 1024 or nothing fits: two kernels per order (sweep_large.cu), plain R layout
  bool sweep_gemm = false;       // large batches: two GEMM launches per order (sweep_gemm.cu), plain R layout
  double2* d_xbuf = nullptr;     // sweep_large: x_s of every map [B][+-][L]
  double2* d_rres = nullptr;     // sweep_large refinement: residual [B][L][+-]
  double* d_at = nullptr;        // refinement: the blocks A_m themselves, tiled like X (offsets of X)
  int refine = 0;                // iterative-refinement steps per order in sweep_large (default 1 for L > 512)
  bool inv_ready = false;        // inverse buffers allocated
  // breadth-first factorisation (factor_bf.cu) of every order
  BfRange bf_full;               // the non-windowed range (every order)
  // Split factorisation (factor.cu): the orders are cut into ranges (high orders first);
  // each range is its own latency-bound chain of panel steps on its own stream, so the
  // blocked sweep can start on the high orders (cheap to factor, first to be swept) while the
  // lower ranges are still being factored.  Range boundaries are sweep block boundaries.
  static constexpr int kFactorRanges = 4;
  BfRange bf_rng[kFactorRanges];            // [0] = the highest orders ... [n-1] = the lowest (on the caller's stream)
  int n_frng = 0;                           // 0: not prepared
  cudaStream_t s_f[kFactorRanges] = {};     // streams of ranges 0 .. n-2
  cudaEvent_t ev_f[kFactorRanges] = {};     // range r done (r < n-1)
  cudaEvent_t ev_fstart = nullptr;
  bool fsplit_active = false;               // the last launch_factor ran split
  bool sweep_waits_ranges = false;          // blocked sweep: wait for each range's event at its first block
  int num_sms = 0;
  bool need_norms = true;        // this call checks conditioning (check=True): factor kernels accumulate norms
  int64_t* d_bf_off = nullptr;   // [L+1] offsets of the E / R panels (NB x lde(n) per order)
  double* d_bf_e = nullptr;
  double* d_bf_e2 = nullptr;     // the second panel's E of a paired step
  double* d_bf_r = nullptr;      // two R buffers of bf_r_half doubles (alternating steps)
  int64_t bf_r_half = 0;
  double* d_bf_d = nullptr;      // NB x NB diagonal-block inverses
  // windowed forward (window.cu): factor storage for all orders does not fit HBM
  bool windowed = false;
  std::vector<FwdWindow> windows;  // descending in m
  float last_factor_ms = 0.f, last_sweep_ms = 0.f;
  // spin-weighted transforms (spin.cu): the two most recently used spins
  std::vector<SpinState*> spins;
  double2* d_spin_xbuf = nullptr;  // [B][+-][L] solved coefficients of the current order

  // ---- per-call workspaces (sized for max_batch) ----
  double* d_fpack = nullptr;  // inverse: packed coefficients [pos(m,l)][4B]
  double* d_g = nullptr;      // inverse: G [m][k][4B]
  double2* d_r = nullptr;     // forward: ring spectra, team-major [team][pos(m,k-m)][2][G] (common.cuh r_index)
  double2* d_in = nullptr;    // device staging of host inputs  [B][L^2]
  double2* d_out = nullptr;   // device staging of host outputs [B][L^2]
  double2* d_z1 = nullptr;    // real maps (OSPH_REAL): paired complex maps [ceil(B/2)][L^2]
  double2* d_z2 = nullptr;

  // stage events: inverse 0 pack 1 synth 2 ring 3; forward ring 4-5, factor 6-7, sweep 8-9
  cudaEvent_t ev[10] = {};
  // host-buffer calls: copies on their own streams, overlapped with compute chunk by chunk
  static constexpr int kIoChunks = 4;
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[kIoChunks] = {}, ev_done[kIoChunks] = {}, ev_start = nullptr, ev_out = nullptr;
  cudaEvent_t ev_sweep_done = nullptr;  // last forward's sweep: the factor buffers are free again
  bool have_sweep_ev = false;
  bool have_inv = false, have_fwd = false;
};

// Saves the calling thread's current device and restores it on scope exit, so
// an entry point that switches to the plan's device leaves the caller's
// device (e.g. torch's current device) untouched.
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaGetLastError();  // a failed call earlier on this thread must not leak into this one's launch checks
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Orders this plan factors: every order unless osph_plan_shard gave it a block.
inline void own_orders(const osph_plan* p, int& lo, int& hi) {
  if (p->shard_mode && p->own_m_hi >= 0) {
    lo = p->own_m_lo;
    hi = p->own_m_hi;
  } else {
    lo = 0;
    hi = p->L - 1;
  }
}

// last-error plumbing (plan.cu)
void osph_set_error(const std::string& msg);

// plan.cu internals shared with shard.cu
int plan_create_one(int L, const double* thetas, int max_batch, int device, osph_plan** out);
void plan_free(osph_plan* p);
int ensure_io(osph_plan* p);
int ensure_inverse(osph_plan* p);
int ensure_forward(osph_plan* p);
int check_call(osph_plan* p, int B, const void* a, void* b, int kind);
int inverse_enqueue(osph_plan* p, int B, const void* flm, void* samples, int kind);
// shard.cu: sharded stages and multi-device plans
int forward_stage_enqueue(osph_plan* p, int stages, int B, const void* samples, void* flm);
int forward_check(osph_plan* p, int check, osph_stats* stats);
int group_create(int L, const double* thetas, int max_batch, int ndev, const int* devs, osph_plan** out);
int group_inverse(osph_plan* p, int B, const void* flm, void* samples, int kind);
int group_forward(osph_plan* p, int B, const void* samples, void* flm, int kind, int check, osph_stats* stats);

// ---- launchers (each returns cudaError_t of the launch) ----
cudaError_t launch_tables(osph_plan* p);
cudaError_t launch_legendre_block(osph_plan* p, int m, double* out, int64_t ld);  // tables.cu
cudaError_t launch_ring_inverse(osph_plan* p, int B, double2* samples);    // ringdft.cu
// maps [bofs, bofs + nb) of a batch of B (nb < 0: all B); plain: R in the [map][pos][+-] layout
cudaError_t launch_ring_forward(osph_plan* p, int B, const double2* samples, int bofs = 0, int nb = -1,
                                bool plain = false);  // ringdft.cu
cudaError_t launch_pack(osph_plan* p, int B, const double2* flm);          // synth.cu
cudaError_t launch_synth(osph_plan* p, int B);                             // synth.cu
cudaError_t launch_factor(osph_plan* p, cudaStream_t st = nullptr);  // factor.cu: every order, breadth-first
cudaError_t launch_sweep(osph_plan* p, int B, double2* flm);               // sweep.cu
int sweep_maps_per_team(osph_plan* p, int B);
cudaError_t launch_sweep_large(osph_plan* p, int B, double2* flm);  // sweep_large.cu
cudaError_t launch_sweep_gemm(osph_plan* p, int B, double2* flm);   // sweep_gemm.cu
// sweep_block.cu; maps b0 .. b0 + B - 1 of the spectra, flm = the first of those maps
cudaError_t launch_sweep_blocked(osph_plan* p, int B, double2* flm, int b0 = 0);
int ensure_sweep_blocked(osph_plan* p);                               // sweep_block.cu: scratch buffers
cudaError_t launch_factor_bf(osph_plan* p, int m_first, int m_last, cudaStream_t st);  // factor_bf.cu
cudaError_t bf_prepare(osph_plan* p, int m_first, int m_last, BfRange* r);               // factor_bf.cu
cudaError_t bf_run(osph_plan* p, const BfRange& r, cudaStream_t st, const BfOffsets& o); // factor_bf.cu
cudaError_t bf_generate(osph_plan* p, const BfRange& r, cudaStream_t st, const BfOffsets& o, bool with_at);
cudaError_t bf_step(osph_plan* p, const BfRange& r, int sidx, cudaStream_t st, const BfOffsets& o, bool fused_r);
int64_t bf_panel_doubles(int n);
int64_t bf_diag_doubles(int orders);
cudaError_t launch_sweep_large_range(osph_plan* p, int B, double2* flm, int s_hi, int s_lo, const int64_t* xt_off,
                                     const int64_t* pb_off);  // sweep_large.cu
int discover_pivots(osph_plan* p);  // pivots.cu: the grid's pivot order (once per grid), host-blocking
int alloc_factor_storage(osph_plan* p);                        // window.cu
void spin_free(osph_plan* p);                                  // spin.cu
int ensure_spectra(osph_plan* p);                              // plan.cu: the ring spectra buffer d_r
void free_windows(osph_plan* p);                               // window.cu
cudaError_t forward_windows(osph_plan* p, int B, double2* flm);  // window.cu: factor + sweep per window
// window.cu, staged: factor window 0 only / sweep every window (factoring windows >= 1 before their sweep)
cudaError_t forward_windows_factor_first(osph_plan* p);
cudaError_t forward_windows_sweep(osph_plan* p, int B, double2* flm);
void window_times(osph_plan* p);                               // window.cu
cudaError_t launch_kappa(osph_plan* p, cudaStream_t st);       // factor.cu
cudaError_t launch_ring_pair(int n, int m, const double2* v, double2* out, cudaStream_t st);  // ringdft.cu
