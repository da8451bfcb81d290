// sweep_gemm.cu -- the order-peeling sweep for large batches (the "batched
// DMMA per-order solve" of BASELINE configs[2]).
//
// Same recurrence as sweep.cu / sweep_large.cu (transform.py:436-467): for
// s = L-1 .. 0, x_s = X_s P [g_+s, (-1)^s g_-s] for every map, then the
// corrections G = Pb_s x_s of rings k < s go to their alias bins.  With many
// maps each order is a real GEMM -- (n x n) x (n x 4B) for the solve and
// (s x n) x (n x 4B) for the corrections -- so each order runs as two
// fp64 tensor-core GEMM launches over the whole GPU instead of the persistent
// per-team kernel (whose teams no longer fit the GPU at once for large B).
// Tiles: 16 rows x 64 columns (16 maps x {+,-} x {re, im}) per CTA (twice
// the CTAs of 32-row tiles: measured 14.3 -> 12.4 ms at config 3), K in
// 32-wide chunks in a 3-stage 16-byte cp.async ring; A operands are the
// chunk-major 8-row tiles the factorisation writes (each 8-row x 32-k piece
// is one contiguous 2 KB run), B operands come straight from R / xbuf.
#include "plan.cuh"

#define SG_THREADS 256
#ifndef SG_TM
#define SG_TM 16   // rows per CTA (16: twice the CTAs of 32 at these per-order GEMM sizes)
#endif
#define SG_MAPS 16 // maps per CTA (64 real columns)
#define SG_KC 32

__device__ __forceinline__ uint32_t sg_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sg_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sg_smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void sg_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

struct SgStage {
  double a[SG_TM / 8][SG_KC][8];          // row tiles as stored: [k][row % 8]
  double b[SG_MAPS][SG_KC][4];            // [map][k][+re, +im, -re, -im]
};

// MODE 0: solve (A = X_s tiles, rows = degrees, K = rings, B = R slab of order s)
// MODE 1: corrections (A = Pb_s tiles, rows = rings k < s, K = degrees, B = xbuf)
template <int N>
__device__ __forceinline__ void sg_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int MODE, int NS>
__global__ void __launch_bounds__(SG_THREADS) k_sweep_gemm(int L, int s, int B, const double* __restrict__ atiles,
                                                           const int64_t* __restrict__ a_off,
                                                           const double* __restrict__ w_all, double2* __restrict__ R,
                                                           double2* __restrict__ xbuf, double2* __restrict__ flm) {
  extern __shared__ __align__(16) unsigned char sg_raw[];
  SgStage* st = reinterpret_cast<SgStage*>(sg_raw);
  const int n = L - s;
  const int M = MODE == 0 ? n : s;            // output rows
  const int nrt = MODE == 0 ? (n + 7) >> 3 : (s + 7) >> 3;
  const int rt0 = blockIdx.x * (SG_TM / 8);   // first 8-row tile
  const int b0 = blockIdx.y * SG_MAPS;
  const double* A = atiles + __ldg(a_off + s);
  const int64_t npos = (int64_t)L * (L + 1) / 2, p0 = packed_pos(L, s, 0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int nch = (n + SG_KC - 1) / SG_KC;

  auto load = [&](int buf, int c) {
    SgStage& S = st[buf];
    // A: SG_TM / 8 row tiles x 2 KB, contiguous within chunk c (zero past the last tile)
    for (int i = tid; i < (SG_TM / 8) * 128; i += SG_THREADS) {  // 128 16-byte pieces per tile
      const int t = i >> 7, q = i & 127;
      double* dst = &S.a[t][0][0] + 2 * q;
      if (rt0 + t < nrt) sg_cp16(dst, A + ((int64_t)c * nrt + rt0 + t) * 256 + 2 * q);
      else *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
    }
    // B: per map, 32 K-entries x {+, -} complex
    for (int i = tid; i < SG_MAPS * SG_KC * 2; i += SG_THREADS) {
      const int mp = i / (SG_KC * 2), rem = i % (SG_KC * 2), k = rem >> 1, slot = rem & 1;
      const int kk = c * SG_KC + k, b = b0 + mp;
      double* dst = &S.b[mp][k][2 * slot];
      if (kk < n && b < B) {
        const double2* src = MODE == 0 ? R + ((int64_t)b * npos + p0 + kk) * 2 + slot
                                       : xbuf + ((int64_t)b * 2 + slot) * L + kk;
        sg_cp16(dst, src);
      } else {
        *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
      }
    }
    sg_commit();
  };

  // warp tile: rows (warp & 1) * (SG_TM / 2) .. (RB blocks of 8), columns (warp >> 1) * 16 .. +16 (2 blocks)
  constexpr int RB = SG_TM / 16;
  const int wr = (warp & 1) * (SG_TM / 2), wc = (warp >> 1) * 16;
  double acc[RB][2][2];
#pragma unroll
  for (int i = 0; i < RB; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // NS-stage cp.async ring: chunks c+1 .. c+NS-1 in flight while chunk c multiplies
  // (empty commit groups past the last chunk keep the group count uniform)
#pragma unroll
  for (int c = 0; c < NS - 1; ++c) {
    if (c < nch) load(c, c);
    else sg_commit();
  }
  for (int c = 0; c < nch; ++c) {
    sg_wait<NS - 2>();
    __syncthreads();  // chunk c visible to all; stage (c - 1) % NS free
    if (c + NS - 1 < nch) load((c + NS - 1) % NS, c + NS - 1);
    else sg_commit();
    const SgStage& S = st[c % NS];
#pragma unroll
    for (int k0 = 0; k0 < SG_KC; k0 += 4) {
      double a[RB], b[2];
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int row = wr + 8 * i + g;
        a[i] = S.a[row >> 3][k0 + tq][row & 7];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = wc + 8 * j + g;  // map col >> 2, component col & 3
        b[j] = S.b[col >> 2][k0 + tq][col & 3];
      }
#pragma unroll
      for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }

  const double sg = (s & 1) ? -1.0 : 1.0;
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    const int row = rt0 * 8 + wr + 8 * i + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int col = wc + 8 * j + 2 * tq;  // even: (re, im) of one (map, slot)
      const int mp = col >> 2, slot = (col >> 1) & 1, b = b0 + mp;
      if (b >= B) continue;
      double vr = acc[i][j][0], vi = acc[i][j][1];
      if (MODE == 0) {
        // late ring's column (zeroed in X tiles): + w[row] * rhs[0]
        const double w = __ldg(w_all + (int64_t)s * uw_ld(L) + row);
        const double2 g0 = R[((int64_t)b * npos + p0) * 2 + slot];
        vr = fma(w, g0.x, vr);
        vi = fma(w, g0.y, vi);
        if (slot) {
          vr *= sg;
          vi *= sg;
        }
        const double2 x = make_double2(vr, vi);
        xbuf[((int64_t)b * 2 + slot) * L + row] = x;
        const int64_t ell = s + row;
        double2* f = flm + (int64_t)b * L * L + ell * ell + ell;
        if (slot == 0) f[s] = x;
        else if (s > 0) f[-s] = x;
      } else {
        // G_-s carries (-1)^s; alias target of ring k = row (transform.py:459-463)
        if (slot) {
          vr *= sg;
          vi *= sg;
        }
        const int k = row, nk = 2 * k + 1, rr = s % nk;
        int tm, ts;
        if (rr == 0) {
          tm = 0;
          ts = 0;
        } else if (rr <= k) {
          tm = rr;
          ts = slot;
        } else {
          tm = nk - rr;
          ts = slot ^ 1;
        }
        double2* rp = R + ((int64_t)b * npos + packed_pos(L, tm, k - tm)) * 2 + ts;
        atomicAdd(&rp->x, -vr);  // r == 0 sends both tones to bin 0: reductions
        atomicAdd(&rp->y, -vi);
      }
    }
  }
}

template <int NS>
static cudaError_t sweep_gemm_run(osph_plan* p, int B, double2* flm) {
  const int L = p->L;
  const size_t smem = NS * sizeof(SgStage);
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_sweep_gemm<0, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_sweep_gemm<1, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  const int ny = (B + SG_MAPS - 1) / SG_MAPS;
  for (int s = L - 1; s >= 0; --s) {
    const int n = L - s;
    k_sweep_gemm<0, NS><<<dim3((n + SG_TM - 1) / SG_TM, ny), SG_THREADS, smem, p->stream>>>(
        L, s, B, p->d_xt, p->d_xt_off, p->d_w, p->d_r, p->d_xbuf, flm);
    if (s >= 1)
      k_sweep_gemm<1, NS><<<dim3((s + SG_TM - 1) / SG_TM, ny), SG_THREADS, smem, p->stream>>>(
          L, s, B, p->d_pbelow, p->d_pb_off, p->d_w, p->d_r, p->d_xbuf, flm);
  }
  p->launches += 2 * L - 1;
  return cudaGetLastError();
}

// cp.async stages of the K loop (OSPH_SG_STAGES=2|3|4).  Config 3 sweep:
// 13.06 / 12.24 / 12.34 ms for 2 / 3 / 4 stages -- the loop is bound by the
// L2 reads of the B chunks (every row-tile CTA re-reads them), not latency
cudaError_t launch_sweep_gemm(osph_plan* p, int B, double2* flm) {
  static const int ns = getenv("OSPH_SG_STAGES") ? atoi(getenv("OSPH_SG_STAGES")) : 3;
  if (ns == 2) return sweep_gemm_run<2>(p, B, flm);
  if (ns == 3) return sweep_gemm_run<3>(p, B, flm);
  return sweep_gemm_run<4>(p, B, flm);
}
