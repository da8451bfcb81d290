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
// Tiles: 64 rows x 16 columns (4 maps x {+,-} x {re, im}) per CTA by
// default (launch_sweep_gemm lists the measured shapes), K in 32-wide
// chunks in a 4-stage 16-byte cp.async ring; A operands are the
// chunk-major 8-row tiles the factorisation writes (each 8-row x 32-k piece
// is one contiguous 2 KB run), B operands come straight from R / xbuf.
#include "plan.cuh"

#define SG_THREADS 256
#define SG_KC 32

__device__ __forceinline__ uint32_t sg_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sg_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sg_smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void sg_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

// CTA tile: TM rows x MAPS maps (4 real columns per map)
template <int TM, int MAPS>
struct SgStage {
  double a[TM / 8][SG_KC][8];          // row tiles as stored: [k][row % 8]
  double b[MAPS][SG_KC][4];            // [map][k][+re, +im, -re, -im]
};

// MODE 0: solve (A = X_s tiles, rows = degrees, K = rings, B = R slab of order s)
// MODE 1: corrections (A = Pb_s tiles, rows = rings k < s, K = degrees, B = xbuf)
template <int N>
__device__ __forceinline__ void sg_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int MODE, int NS, int TM, int MAPS>
__global__ void __launch_bounds__(SG_THREADS) k_sweep_gemm(int L, int s, int B, const double* __restrict__ atiles,
                                                           const int64_t* __restrict__ a_off,
                                                           const double* __restrict__ w_all, double2* __restrict__ R,
                                                           double2* __restrict__ xbuf, double2* __restrict__ flm) {
  pdl_start();
  extern __shared__ __align__(16) unsigned char sg_raw[];
  using Stage = SgStage<TM, MAPS>;
  Stage* st = reinterpret_cast<Stage*>(sg_raw);
  const int n = L - s;
  const int M = MODE == 0 ? n : s;            // output rows
  const int nrt = MODE == 0 ? (n + 7) >> 3 : (s + 7) >> 3;
  const int rt0 = blockIdx.x * (TM / 8);   // first 8-row tile
  const int b0 = blockIdx.y * MAPS;
  const double* A = atiles + __ldg(a_off + s);
  const int64_t npos = (int64_t)L * (L + 1) / 2, p0 = packed_pos(L, s, 0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int nch = (n + SG_KC - 1) / SG_KC;

  auto load = [&](int buf, int c) {
    Stage& S = st[buf];
    // A: TM / 8 row tiles x 2 KB, contiguous within chunk c (zero past the last tile)
    for (int i = tid; i < (TM / 8) * 128; i += SG_THREADS) {  // 128 16-byte pieces per tile
      const int t = i >> 7, q = i & 127;
      double* dst = &S.a[t][0][0] + 2 * q;
      if (rt0 + t < nrt) sg_cp16(dst, A + ((int64_t)c * nrt + rt0 + t) * 256 + 2 * q);
      else *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
    }
    // B: per map, 32 K-entries x {+, -} complex
    for (int i = tid; i < MAPS * SG_KC * 2; i += SG_THREADS) {
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

  // warps: WCG column groups of 16 (2 blocks of 8) x WRG row groups of RB blocks of 8
  constexpr int WCG = MAPS / 4, WRG = 8 / WCG, RB = TM / (8 * WRG);
  static_assert(WCG * WRG == 8 && RB >= 1 && RB * 8 * WRG == TM, "CTA tile does not map onto 8 warps");
  const int wr = (warp % WRG) * (TM / WRG), wc = (warp / WRG) * 16;
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
    const Stage& S = st[c % NS];
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
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (row >= M) continue;
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
        if (rr == 0) {  // bin 0: -tones into order 0's unused - slot (no racing REDs; folded at s = 0)
          tm = 0;
          ts = slot;
        } else if (rr <= k) {
          tm = rr;
          ts = slot;
        } else {
          tm = nk - rr;
          ts = slot ^ 1;
        }
        double2* rp = R + ((int64_t)b * npos + packed_pos(L, tm, k - tm)) * 2 + ts;
        atomicAdd(&rp->x, -vr);
        atomicAdd(&rp->y, -vi);
      }
    }
  }
}

// R[b][pos(0, k)][+] += R[b][pos(0, k)][-] for every ring k (plain layout).
__global__ void k_fold_order0(int L, double2* __restrict__ R) {
  pdl_start();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  double2* rp = R + ((int64_t)blockIdx.y * npos + k) * 2;  // pos(0, k) = k
  rp[0] = make_double2(rp[0].x + rp[1].x, rp[0].y + rp[1].y);
}

template <int NS, int TM, int MAPS>
static cudaError_t sweep_gemm_run(osph_plan* p, int B, double2* flm) {
  const int L = p->L;
  const size_t smem = NS * sizeof(SgStage<TM, MAPS>);
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_sweep_gemm<0, NS, TM, MAPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_sweep_gemm<1, NS, TM, MAPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem)) != cudaSuccess)
    return e;
  const int ny = (B + MAPS - 1) / MAPS;
  for (int s = L - 1; s >= 0; --s) {
    const int n = L - s;
    if (s == 0) {  // order 0: fold the - slot (bin-0 -tone corrections) into the + slot
      launch_pdl(k_fold_order0, dim3((L + 127) / 128, B), dim3(128), 0, p->stream, L, p->d_r);
      p->launches++;
    }
    launch_pdl(k_sweep_gemm<0, NS, TM, MAPS>, dim3((n + TM - 1) / TM, ny), dim3(SG_THREADS), smem, p->stream, L, s,
               B, (const double*)p->d_xt, (const int64_t*)p->d_xt_off, (const double*)p->d_w, p->d_r, p->d_xbuf, flm);
    if (s >= 1)
      launch_pdl(k_sweep_gemm<1, NS, TM, MAPS>, dim3((s + TM - 1) / TM, ny), dim3(SG_THREADS), smem, p->stream, L,
                 s, B, (const double*)p->d_pbelow, (const int64_t*)p->d_pb_off, (const double*)p->d_w, p->d_r,
                 p->d_xbuf, flm);
  }
  p->launches += 2 * L - 1;
  return cudaGetLastError();
}

// CTA tile 64 rows x 4 maps, 4 cp.async stages of the K loop.  The loop is
// bound by the L2 reads of the operand chunks -- every CTA of a map group
// re-reads the B chunk, every map group the A chunk -- so the tile shape
// decides.  Measured alternatives (config 3 sweep, ms; removed): 16x16 13.06 /
// 12.24 / 12.34 with 2 / 3 / 4 stages; 32x8 11.25 / 10.99 / 11.12 with 3 / 4 /
// 6; 64x4 11.07 / 10.79 / 12.34 with 3 / 4 / 6; 64x8 13.21; 32x16 14.02.
cudaError_t launch_sweep_gemm(osph_plan* p, int B, double2* flm) { return sweep_gemm_run<4, 64, 4>(p, B, flm); }
