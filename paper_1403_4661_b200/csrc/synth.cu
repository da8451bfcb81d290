// synth.cu -- inverse Legendre synthesis G_(+-m)(theta_k) = sum_l P_lm(theta_k) f_l(+-m).
//
// Reference: _synthesis_g / _g_accumulate (pkg/src/optisph/transform.py:143-201,
// 310-331): for every ring i and order m the recurrence of
// legendre.py:64-96 is fused with a four-stream dot product
// [Re f_m, Im f_m, Re f_-m, Im f_-m].  Here the 4 streams of all B maps form
// the C = 4B columns of a per-order product
//     G_m[k][c] = sum_l P_m[k][l] * F_m[l][c]
// with P_m generated on the fly by the upward recurrence (never stored) and
// started at the precomputed first in-range degree ls(m,k) (tables.cu), so
// the hot loops carry no rescaling branches.  2*pi and (-1)^m are applied by
// the ring kernels.  Two kernels:
//   * k_synth_fma  (C <= 8): one thread per (ring, order), FMA pipe;
//   * k_synth_dmma (C >= 16): 64x64 output tiles on fp64 tensor cores
//     (mma.sync m8n8k4 -> SASS DMMA.8x8x4); P tiles generated into shared
//     memory by two warps while the others stage F.
#include <cstdlib>

#include "plan.cuh"

// flm [B][L^2] complex -> F [pos(m, l-m)][4B] doubles:
// c = 4b + {0: Re f_lm, 1: Im f_lm, 2: Re f_l,-m, 3: Im f_l,-m}.
__global__ void k_pack(int L, int B, const double2* __restrict__ flm, double* __restrict__ F) {
  const int m = blockIdx.y;
  const int n = L - m;
  const int64_t total = (int64_t)n * B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(t % B);
    const int i = (int)(t / B);
    const int64_t l = m + i;
    const double2* f = flm + (int64_t)b * L * L + l * l + l;
    const double2 fp = __ldg(f + m);
    const double2 fn = __ldg(f - m);
    double4* dst = reinterpret_cast<double4*>(F + (packed_pos(L, m, i) * B + b) * 4);
    *dst = make_double4(fp.x, fp.y, fn.x, fn.y);
  }
}

cudaError_t launch_pack(osph_plan* p, int B, const double2* flm) {
  const int L = p->L;
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(((int64_t)L * B + 255) / 256, 64)), L);
  k_pack<<<grid, 256, 0, p->stream>>>(L, B, flm, p->d_fpack);
  p->launches++;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// FMA path: C <= 8 columns (B <= 2 maps).

#define SYN_FMA_THREADS 128
#define SYN_FMA_CHUNK 256

template <int C>
__global__ void __launch_bounds__(SYN_FMA_THREADS) k_synth_fma(
    int L, int nr, const double* __restrict__ costh, const double2* __restrict__ rec, const int* __restrict__ ls_tab,
    const double2* __restrict__ pstart, const int* __restrict__ ring_order, const double* __restrict__ F,
    double* __restrict__ G) {
  __shared__ double Fs[SYN_FMA_CHUNK * C];
  __shared__ double2 Rs[SYN_FMA_CHUNK];
  const int m = blockIdx.y;
  const int idx = blockIdx.x * SYN_FMA_THREADS + threadIdx.x;
  const bool active = idx < nr;  // ring_order lists the nr rings to synthesise
  const int k = active ? ring_order[idx] : 0;
  const int64_t t = (int64_t)m * L + k;
  int ls = active ? ls_tab[t] : L;
  double2 pp = active ? pstart[t] : make_double2(0.0, 0.0);
  double p0 = pp.x, p1 = pp.y;
  const double x = costh[k];
  double acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.0;
  // block-wide first useful degree
  int lmin = ls;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
  __shared__ int wmin[SYN_FMA_THREADS / 32];
  if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = lmin;
  __syncthreads();
  lmin = wmin[0];
  for (int w = 1; w < SYN_FMA_THREADS / 32; ++w) lmin = min(lmin, wmin[w]);
  const double* Fm = F + packed_pos(L, m, 0) * C;
  const double2* recm = rec + packed_pos(L, m, 0);
  for (int cs = lmin; cs < L; cs += SYN_FMA_CHUNK) {
    const int ce = min(L, cs + SYN_FMA_CHUNK);
    __syncthreads();
    for (int i = threadIdx.x; i < (ce - cs) * C; i += SYN_FMA_THREADS) Fs[i] = __ldg(Fm + (int64_t)(cs - m) * C + i);
    for (int i = threadIdx.x; i < ce - cs; i += SYN_FMA_THREADS) Rs[i] = __ldg(recm + (cs - m) + i);
    __syncthreads();
    for (int l = max(cs, ls); l < ce; ++l) {
      const int j = l - cs;
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = fma(p1, Fs[j * C + c], acc[c]);
      const double2 ar = Rs[j];
      const double nxt = fma(x, p1, -ar.x * p0) * ar.y;
      p0 = p1;
      p1 = nxt;
    }
  }
  if (active) {
    double* g = G + ((int64_t)m * L + k) * C;
#pragma unroll
    for (int c = 0; c < C; ++c) g[c] = acc[c];
  }
}

// ---------------------------------------------------------------------------
// DMMA path: C >= 16.  Block tile 64 rings x TN columns (TN = 64/128/256: the
// Legendre block generated for a tile is reused by TN columns), K chunks of 16
// degrees, double
// buffered: two warps run the ring recurrences of the next chunk and every
// thread streams its share of the next F chunk with cp.async while the chunk
// in hand is multiplied on the tensor cores.

#define SYN_TM 64
#define SYN_TK 16
#define SYN_THREADS 256
#define SYN_PAD 4  // row pitch = 4 mod 16 doubles: conflict-free DMMA fragment loads

__device__ __forceinline__ void syn_cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

template <int TN>
__global__ void __launch_bounds__(SYN_THREADS, TN > 128 ? 1 : 2) k_synth_dmma(
    int L, int nr, int C, const double* __restrict__ costh, const double2* __restrict__ rec,
    const int* __restrict__ ls_tab, const double2* __restrict__ pstart, const int* __restrict__ ring_order,
    const double* __restrict__ F, double* __restrict__ G) {
  constexpr int NT = TN / 16;  // 8-column tiles per warp (warp tile 16 rows x TN/2 columns)
  extern __shared__ __align__(16) double syn_smem[];
  double(*Ps)[SYN_TK][SYN_TM + SYN_PAD] = reinterpret_cast<double(*)[SYN_TK][SYN_TM + SYN_PAD]>(syn_smem);
  double(*Fs)[SYN_TK][TN + SYN_PAD] =
      reinterpret_cast<double(*)[SYN_TK][TN + SYN_PAD]>(syn_smem + 2 * SYN_TK * (SYN_TM + SYN_PAD));
  __shared__ int s_lmin[2];
  const int m = blockIdx.z;
  const int row0 = blockIdx.y * SYN_TM;
  const int col0 = blockIdx.x * TN;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;

  // generator state: threads 0..63 own one ring each
  int ls = L, kring = 0;
  double p0 = 0.0, p1 = 0.0, x = 0.0;
  if (tid < SYN_TM) {
    const int r = row0 + tid;
    if (r < nr) {  // ring_order lists the nr rings to synthesise
      kring = ring_order[r];
      const int64_t t = (int64_t)m * L + kring;
      ls = ls_tab[t];
      const double2 pp = pstart[t];
      p0 = pp.x;
      p1 = pp.y;
      x = costh[kring];
    }
  }
  if (tid < 2) s_lmin[tid] = L;
  __syncthreads();
  if (tid < SYN_TM) atomicMin(&s_lmin[0], ls);
  __syncthreads();
  const int lstart = s_lmin[0];
  // chunk grid aligned to m so F loads stay aligned to the packed order start
  const int kfirst = m + ((lstart - m) / SYN_TK) * SYN_TK;
  const double* Fm = F + packed_pos(L, m, 0) * (int64_t)C;
  const double2* recm = rec + packed_pos(L, m, 0);

  const int wr = (warp & 3) * 16;
  const int wc = (warp >> 2) * (TN / 2);
  double acc[2][NT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto produce = [&](int buf, int ks) {
    // F chunk: 16 degrees x TN columns, 16-byte async copies (zero outside)
    for (int i = tid; i < SYN_TK * TN / 2; i += SYN_THREADS) {
      const int j = i / (TN / 2);
      const int c2 = (i % (TN / 2)) * 2;
      const int l = ks + j;
      const int c = col0 + c2;
      double* dst = &Fs[buf][j][c2];
      if (l < L && c < C) syn_cp_async16(dst, Fm + (int64_t)(l - m) * C + c);  // C is a multiple of 4
      else *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    if (tid < SYN_TM) {
      // recurrence factors of the chunk fetched 8 at a time (independent loads,
      // one exposed latency per batch instead of one per degree)
#pragma unroll
      for (int j8 = 0; j8 < SYN_TK; j8 += 8) {
        double2 ar[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int l = ks + j8 + u;
          ar[u] = l < L ? __ldg(recm + (l - m)) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int l = ks + j8 + u;
          double v = 0.0;
          if (l < L && l >= ls) {
            v = p1;
            const double nxt = fma(x, p1, -ar[u].x * p0) * ar[u].y;
            p0 = p1;
            p1 = nxt;
          }
          Ps[buf][j8 + u][tid] = v;
        }
      }
    }
  };

  int buf = 0;
  if (kfirst < L) produce(0, kfirst);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  for (int ks = kfirst; ks < L; ks += SYN_TK) {
    if (ks + SYN_TK < L) produce(buf ^ 1, ks + SYN_TK);
#pragma unroll
    for (int kk = 0; kk < SYN_TK; kk += 4) {
      double a[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = Ps[buf][kk + tq][wr + i * 8 + g];
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const double b = Fs[buf][kk + tq][wc + j * 8 + g];
#pragma unroll
        for (int i = 0; i < 2; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b);
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    buf ^= 1;
  }
  // store: C fragment rows = ring positions, cols = 2tq, 2tq+1
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = row0 + wr + i * 8 + g;
    if (r >= nr) continue;
    const int k = ring_order[r];
    double* grow = G + ((int64_t)m * L + k) * C;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int c = col0 + wc + j * 8 + 2 * tq;
      if (c < C) *reinterpret_cast<double2*>(grow + c) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
}

template <int TN>
static cudaError_t launch_synth_tn(osph_plan* p, int C) {
  const int L = p->L;
  const size_t smem = sizeof(double) * 2 * SYN_TK * ((SYN_TM + SYN_PAD) + (TN + SYN_PAD));
  cudaError_t e = cudaFuncSetAttribute(k_synth_dmma<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((C + TN - 1) / TN, (p->inv_nr + SYN_TM - 1) / SYN_TM, L);
  k_synth_dmma<TN><<<grid, SYN_THREADS, smem, p->stream>>>(L, p->inv_nr, C, p->d_cos, p->d_rec, p->d_ls,
                                                           p->d_pstart, p->d_inv_ring_order, p->d_fpack, p->d_g);
  return cudaGetLastError();
}

cudaError_t launch_synth(osph_plan* p, int B) {
  const int L = p->L;
  const int C = 4 * B;
  if (C <= 8) {
    dim3 grid((p->inv_nr + SYN_FMA_THREADS - 1) / SYN_FMA_THREADS, L);
    if (C == 4)
      k_synth_fma<4><<<grid, SYN_FMA_THREADS, 0, p->stream>>>(L, p->inv_nr, p->d_cos, p->d_rec, p->d_ls, p->d_pstart,
                                                            p->d_inv_ring_order, p->d_fpack, p->d_g);
    else
      k_synth_fma<8><<<grid, SYN_FMA_THREADS, 0, p->stream>>>(L, p->inv_nr, p->d_cos, p->d_rec, p->d_ls, p->d_pstart,
                                                            p->d_inv_ring_order, p->d_fpack, p->d_g);
  } else {
    // widest column tile that the batch fills at least half of
    static const int tn_env = getenv("OSPH_SYNTH_TN") ? atoi(getenv("OSPH_SYNTH_TN")) : 0;
    const int tn = tn_env ? tn_env : (C > 64 ? 128 : 64);  // measured: 128 beats 256 (1 block/SM) at C = 256
    cudaError_t e = tn == 256 ? launch_synth_tn<256>(p, C) : tn == 128 ? launch_synth_tn<128>(p, C) : launch_synth_tn<64>(p, C);
    if (e != cudaSuccess) return e;
  }
  p->launches++;
  return cudaGetLastError();
}
