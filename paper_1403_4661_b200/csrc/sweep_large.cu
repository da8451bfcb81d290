// sweep_large.cu -- the order-peeling sweep for band limits whose right-hand
// sides do not fit the persistent sweep's shared memory (L > 1024).
//
// Same recurrence as sweep.cu (_forward_spectral, transform.py:436-467, with
// the solve of transform.py:396-406): for s = L-1 .. 0
//   x_s = X_s P [g_+s, (-1)^s g_-s]          (rhs = R[pos(s, 0..n-1)][+-])
//   f_(l, +-s) = x_s                          -> flm, and x_s -> xbuf
//   G_(+-s)(theta_k) = Pb_s[k, :] x_s, k < s  (Pb_s = 2pi Y_ls(theta_k); G_-s carries (-1)^s)
//   R[alias target of (s, k, +-)] -= G        (transform.py:459-463)
// as two kernels per order on the plan stream.  At these sizes one order's
// operands (X_s: n^2 doubles, Pb_s: s n doubles, up to 32 MB at L = 2048) are
// streamed from HBM by the whole GPU, so the step is bandwidth-bound and the
// launch gap (~2-3 us) is small against it; nothing is pipelined across
// orders.  One block per 8-row tile of the operand (tiles as the factor
// kernels store them), one or two maps per block.
#include <cstdlib>

#include "plan.cuh"

#define SL_THREADS 256

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Tile-coalesced variants: one block per 8-row tile, warps split the 32-column
// chunks, lane = column: a lane reads its column's 8 rows as one contiguous
// 64-byte run, so a warp consumes a whole 2 KB tile block per step.
// rhs of map b, ring offset j, slot: R[(b * npos + p0 + j) * 2 + slot]; accumulate: x += X rhs
// (the refinement step, whose rhs is the residual in a scratch with npos = L, p0 = 0)
template <int MB>
__global__ void __launch_bounds__(SL_THREADS) k_sweep_solve_t(int L, int s, int B, const double* __restrict__ xt,
                                                              const int64_t* __restrict__ xt_off,
                                                              const double* __restrict__ w_all,
                                                              const double2* __restrict__ R,
                                                              double2* __restrict__ xbuf, double2* __restrict__ flm,
                                                              int64_t npos, int64_t p0, int accumulate) {
  pdl_start();
  __shared__ double red[SL_THREADS / 32][8][4 * MB];
  const int n = L - s, nrt = (n + 7) >> 3;
  const int rt = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* X = xt + __ldg(xt_off + s);
  const int nch = (n + 31) >> 5;
  for (int b0 = blockIdx.y * MB; b0 < B; b0 += gridDim.y * MB) {
    double acc[8][4 * MB];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4 * MB; ++q) acc[r][q] = 0.0;
    for (int c = warp; c < nch; c += SL_THREADS / 32) {
      const int j = c * 32 + lane;
      if (j < n) {
        const double2* xp = reinterpret_cast<const double2*>(X + ((int64_t)c * nrt + rt) * 256 + lane * 8);
        double xr[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const double2 v = __ldg(xp + h);
          xr[2 * h] = v.x;
          xr[2 * h + 1] = v.y;
        }
#pragma unroll
        for (int q = 0; q < MB; ++q) {
          if (b0 + q < B) {
            const double2* rp = R + ((int64_t)(b0 + q) * npos + p0 + j) * 2;
            const double2 gp = __ldg(rp), gn = __ldg(rp + 1);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              acc[r][4 * q + 0] = fma(xr[r], gp.x, acc[r][4 * q + 0]);
              acc[r][4 * q + 1] = fma(xr[r], gp.y, acc[r][4 * q + 1]);
              acc[r][4 * q + 2] = fma(xr[r], gn.x, acc[r][4 * q + 2]);
              acc[r][4 * q + 3] = fma(xr[r], gn.y, acc[r][4 * q + 3]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4 * MB; ++q) {
        const double v = warp_sum(acc[r][q]);
        if (lane == 0) red[warp][r][q] = v;
      }
    __syncthreads();
    if (threadIdx.x < 8 * MB) {
      const int r = threadIdx.x & 7, q = threadIdx.x >> 3;
      const int row = rt * 8 + r;
      if (row < n && b0 + q < B) {
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        for (int w = 0; w < SL_THREADS / 32; ++w)
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] += red[w][r][4 * q + u];
        const double w = __ldg(w_all + (int64_t)s * uw_ld(L) + row);  // X[:, j*]: the late ring's column
        const double2* rp = R + ((int64_t)(b0 + q) * npos + p0) * 2;
        const double2 gp = rp[0], gn = rp[1];
        const double sg = (s & 1) ? -1.0 : 1.0;
        double2 xp = make_double2(fma(w, gp.x, v[0]), fma(w, gp.y, v[1]));
        double2 xn = make_double2(sg * fma(w, gn.x, v[2]), sg * fma(w, gn.y, v[3]));
        double2* xb = xbuf + ((int64_t)(b0 + q) * 2) * L + row;
        if (accumulate) {
          const double2 op = xb[0], on = xb[L];
          xp = make_double2(op.x + xp.x, op.y + xp.y);
          xn = make_double2(on.x + xn.x, on.y + xn.y);
        }
        xb[0] = xp;
        xb[L] = xn;
        const int64_t ell = s + row;
        double2* f = flm + (int64_t)(b0 + q) * L * L + ell * ell + ell;
        f[s] = xp;
        if (s > 0) f[-s] = xn;
      }
    }
    __syncthreads();
  }
}

// One step of iterative refinement's residual (fixed precision): for ring
// j = k - s of the block, r+ = g+ - A x+,  r- = g- - (-1)^s A x- (so that
// (-1)^s X r- is the correction of x-), A[j][l] = 2pi Y_(s+l),s(theta_k)
// generated by the recurrence from the start table.  One thread per ring.
__global__ void __launch_bounds__(128) k_sweep_resid(int L, int s, int B, const double* __restrict__ costh,
                                                     const double2* __restrict__ rec, const int* __restrict__ ls_tab,
                                                     const double2* __restrict__ pstart,
                                                     const double2* __restrict__ R, const double2* __restrict__ xbuf,
                                                     double2* __restrict__ rres) {
  pdl_start();
  const int n = L - s;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (j >= n || b >= B) return;
  const int k = s + j;
  const int64_t ts = (int64_t)s * L + k;
  const int ls = __ldg(ls_tab + ts);
  const double2 pp = __ldg(pstart + ts);
  double p0 = pp.x, p1 = pp.y;
  const double x = __ldg(costh + k);
  const double2* recs = rec + packed_pos(L, s, 0);
  const double2* xp = xbuf + ((int64_t)b * 2) * L;
  const double2* xn = xp + L;
  double apr = 0.0, api = 0.0, anr = 0.0, ani = 0.0;
  for (int l = max(ls, s); l < L; ++l) {
    const double a = OSPH_TWO_PI * p1;
    const double2 vp = __ldg(xp + (l - s)), vn = __ldg(xn + (l - s));
    apr = fma(a, vp.x, apr);
    api = fma(a, vp.y, api);
    anr = fma(a, vn.x, anr);
    ani = fma(a, vn.y, ani);
    const double2 ar = __ldg(recs + (l - s));
    const double nxt = fma(x, p1, -ar.x * p0) * ar.y;
    p0 = p1;
    p1 = nxt;
  }
  const double sg = (s & 1) ? -1.0 : 1.0;
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  const double2* rp = R + ((int64_t)b * npos + packed_pos(L, s, j)) * 2;
  const double2 gp = rp[0], gn = rp[1];
  double2* o = rres + ((int64_t)b * L + j) * 2;
  o[0] = make_double2(gp.x - apr, gp.y - api);
  o[1] = make_double2(gn.x - sg * anr, gn.y - sg * ani);
}

template <int MB>
__global__ void __launch_bounds__(SL_THREADS) k_sweep_corr_t(int L, int s, int B, const double* __restrict__ pbt,
                                                             const int64_t* __restrict__ pb_off,
                                                             const double2* __restrict__ xbuf,
                                                             double2* __restrict__ R) {
  pdl_start();
  __shared__ double red[SL_THREADS / 32][8][4 * MB];
  const int n = L - s, nrtpb = (s + 7) >> 3;
  const int rt = blockIdx.x;  // rings 8 rt .. 8 rt + 7 (< s)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* Pb = pbt + __ldg(pb_off + s);
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  const int nch = (n + 31) >> 5;
  for (int b0 = blockIdx.y * MB; b0 < B; b0 += gridDim.y * MB) {
    double acc[8][4 * MB];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4 * MB; ++q) acc[r][q] = 0.0;
    for (int c = warp; c < nch; c += SL_THREADS / 32) {
      const int l = c * 32 + lane;
      if (l < n) {
        const double2* pp = reinterpret_cast<const double2*>(Pb + ((int64_t)c * nrtpb + rt) * 256 + lane * 8);
        double pr[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const double2 v = __ldg(pp + h);
          pr[2 * h] = v.x;
          pr[2 * h + 1] = v.y;
        }
#pragma unroll
        for (int q = 0; q < MB; ++q) {
          if (b0 + q < B) {
            const double2 xp = __ldg(xbuf + ((int64_t)(b0 + q) * 2 + 0) * L + l);
            const double2 xn = __ldg(xbuf + ((int64_t)(b0 + q) * 2 + 1) * L + l);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              acc[r][4 * q + 0] = fma(pr[r], xp.x, acc[r][4 * q + 0]);
              acc[r][4 * q + 1] = fma(pr[r], xp.y, acc[r][4 * q + 1]);
              acc[r][4 * q + 2] = fma(pr[r], xn.x, acc[r][4 * q + 2]);
              acc[r][4 * q + 3] = fma(pr[r], xn.y, acc[r][4 * q + 3]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4 * MB; ++q) {
        const double v = warp_sum(acc[r][q]);
        if (lane == 0) red[warp][r][q] = v;
      }
    __syncthreads();
    if (threadIdx.x < 8 * MB) {
      const int r = threadIdx.x & 7, q = threadIdx.x >> 3;
      const int k = rt * 8 + r;
      if (k < s && b0 + q < B) {
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        for (int w = 0; w < SL_THREADS / 32; ++w)
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] += red[w][r][4 * q + u];
        const double sg = (s & 1) ? -1.0 : 1.0;
        const int nk = 2 * k + 1, rr = s % nk;
        int tm, slot_p, slot_n;
        if (rr == 0) {
          tm = 0;
          slot_p = slot_n = 0;
        } else if (rr <= k) {
          tm = rr;
          slot_p = 0;
          slot_n = 1;
        } else {
          tm = nk - rr;
          slot_p = 1;
          slot_n = 0;
        }
        double2* rp = R + ((int64_t)(b0 + q) * npos + packed_pos(L, tm, k - tm)) * 2;
        if (slot_p == slot_n) {  // r == 0: both tones land in bin 0
          rp[0].x -= v[0] + sg * v[2];
          rp[0].y -= v[1] + sg * v[3];
        } else {
          rp[slot_p].x -= v[0];
          rp[slot_p].y -= v[1];
          rp[slot_n].x -= sg * v[2];
          rp[slot_n].y -= sg * v[3];
        }
      }
    }
    __syncthreads();
  }
}

// Residual from the stored block A_s (chunk-major 8-ring tiles, natural ring
// order, written by the factor's generate pass): one block per 8-ring tile,
// the same coalesced pattern as k_sweep_corr_t.  r+ = g+ - A x+,
// r- = g- - (-1)^s A x-.
template <int MB>
__global__ void __launch_bounds__(SL_THREADS) k_sweep_resid_t(int L, int s, int B, const double* __restrict__ at,
                                                              const int64_t* __restrict__ at_off,
                                                              const double2* __restrict__ R,
                                                              const double2* __restrict__ xbuf,
                                                              double2* __restrict__ rres) {
  pdl_start();
  __shared__ double red[SL_THREADS / 32][8][4 * MB];
  const int n = L - s, nrt = (n + 7) >> 3;
  const int rt = blockIdx.x;  // rings s + 8 rt .. s + 8 rt + 7
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* A = at + __ldg(at_off + s);
  const int64_t npos = (int64_t)L * (L + 1) / 2, p0 = packed_pos(L, s, 0);
  const int nch = (n + 31) >> 5;
  for (int b0 = blockIdx.y * MB; b0 < B; b0 += gridDim.y * MB) {
    double acc[8][4 * MB];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4 * MB; ++q) acc[r][q] = 0.0;
    for (int c = warp; c < nch; c += SL_THREADS / 32) {
      const int l = c * 32 + lane;
      if (l < n) {
        const double2* pp = reinterpret_cast<const double2*>(A + ((int64_t)c * nrt + rt) * 256 + lane * 8);
        double ar[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const double2 v = __ldg(pp + h);
          ar[2 * h] = v.x;
          ar[2 * h + 1] = v.y;
        }
#pragma unroll
        for (int q = 0; q < MB; ++q) {
          if (b0 + q < B) {
            const double2 xp = __ldg(xbuf + ((int64_t)(b0 + q) * 2 + 0) * L + l);
            const double2 xn = __ldg(xbuf + ((int64_t)(b0 + q) * 2 + 1) * L + l);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              acc[r][4 * q + 0] = fma(ar[r], xp.x, acc[r][4 * q + 0]);
              acc[r][4 * q + 1] = fma(ar[r], xp.y, acc[r][4 * q + 1]);
              acc[r][4 * q + 2] = fma(ar[r], xn.x, acc[r][4 * q + 2]);
              acc[r][4 * q + 3] = fma(ar[r], xn.y, acc[r][4 * q + 3]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4 * MB; ++q) {
        const double v = warp_sum(acc[r][q]);
        if (lane == 0) red[warp][r][q] = v;
      }
    __syncthreads();
    if (threadIdx.x < 8 * MB) {
      const int r = threadIdx.x & 7, q = threadIdx.x >> 3;
      const int j = rt * 8 + r;
      if (j < n && b0 + q < B) {
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        for (int w = 0; w < SL_THREADS / 32; ++w)
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] += red[w][r][4 * q + u];
        const double sg = (s & 1) ? -1.0 : 1.0;
        const double2* rp = R + ((int64_t)(b0 + q) * npos + p0 + j) * 2;
        const double2 gp = rp[0], gn = rp[1];
        double2* o = rres + ((int64_t)(b0 + q) * L + j) * 2;
        o[0] = make_double2(gp.x - v[0], gp.y - v[1]);
        o[1] = make_double2(gn.x - sg * v[2], gn.y - sg * v[3]);
      }
    }
    __syncthreads();
  }
}

// R must be in the plain [map][pos][+-] layout (maps per team 1, lgG = 0).
cudaError_t launch_sweep_large_range(osph_plan* p, int B, double2* flm, int s_hi, int s_lo, const int64_t* xt_off,
                                     const int64_t* pb_off) {
  const int L = p->L;
  const int mb = B >= 2 ? 2 : 1;
  const int ymaps = (B + mb - 1) / mb;
  // every launch of the chain: programmatic dependent launch (common.cuh)
  const dim3 blk(SL_THREADS);
  const double* xt = p->d_xt;
  const double* wv = p->d_w;
  const double* pbt = p->d_pbelow;
  const double* at = p->d_at;
  for (int s = s_hi; s >= s_lo; --s) {
    const int n = L - s;
    const int64_t npos = (int64_t)L * (L + 1) / 2, p0 = packed_pos(L, s, 0);
    const dim3 gn((n + 7) / 8, ymaps), gs((s + 7) / 8, ymaps);
    auto solve = [&](const double2* rhs, int64_t np, int64_t q0, int acc) {
      if (mb == 2)
        launch_pdl(k_sweep_solve_t<2>, gn, blk, 0, p->stream, L, s, B, xt, xt_off, wv, rhs, p->d_xbuf, flm, np, q0, acc);
      else
        launch_pdl(k_sweep_solve_t<1>, gn, blk, 0, p->stream, L, s, B, xt, xt_off, wv, rhs, p->d_xbuf, flm, np, q0, acc);
      p->launches++;
    };
    solve(p->d_r, npos, p0, 0);
    for (int rstep = 0; rstep < p->refine; ++rstep) {  // x += X (b - A x): fixed-precision refinement
      const double2* r = p->d_r;
      const double2* xb = p->d_xbuf;
      if (p->d_at) {  // stored block (tiled like X)
        if (mb == 2)
          launch_pdl(k_sweep_resid_t<2>, gn, blk, 0, p->stream, L, s, B, at, xt_off, r, xb, p->d_rres);
        else
          launch_pdl(k_sweep_resid_t<1>, gn, blk, 0, p->stream, L, s, B, at, xt_off, r, xb, p->d_rres);
      } else {
        launch_pdl(k_sweep_resid, dim3((n + 127) / 128, B), dim3(128), 0, p->stream, L, s, B, (const double*)p->d_cos,
                   (const double2*)p->d_rec, (const int*)p->d_ls, (const double2*)p->d_pstart, r, xb, p->d_rres);
      }
      solve(p->d_rres, L, 0, 1);
      p->launches++;
    }
    if (s >= 1) {
      const double2* xb = p->d_xbuf;
      if (mb == 2)
        launch_pdl(k_sweep_corr_t<2>, gs, blk, 0, p->stream, L, s, B, pbt, pb_off, xb, p->d_r);
      else
        launch_pdl(k_sweep_corr_t<1>, gs, blk, 0, p->stream, L, s, B, pbt, pb_off, xb, p->d_r);
      p->launches++;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_sweep_large(osph_plan* p, int B, double2* flm) {
  return launch_sweep_large_range(p, B, flm, p->L - 1, 0, p->d_xt_off, p->d_pb_off);
}
