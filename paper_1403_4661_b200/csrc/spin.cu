// spin.cu -- spin-weighted transforms: spin_inverse_sht and
// spin_forward_sht (pkg/src/optisph/transform.py:474-533) over the spin basis
// sY_lm(theta, 0) of legendre.py:223-314.
//
// The control flow is the scalar path's, with one table per SIGNED order
// (the +m and -m blocks differ once s != 0; index u = m + L - 1):
//   inverse  G_(+-m)(theta_k) = sum_(l >= lo) sY_l(+-m)(theta_k) f_l(+-m),
//            lo = max(m, |s|) (k_spin_synth: recurrence generated on the fly
//            from a start table, as synth.cu), then the scalar ring inverse
//            DFTs (fold + Bluestein, ringdft.cu);
//   forward  ring forward DFTs (plain spectra layout), then for m = L-1 .. 0:
//            x_(+-m) = X_(+-m) g_(+-m) (k_spin_solve) and the corrections of
//            the aliased bins of rings k < m, Pb_(+-m) x_(+-m) (k_spin_corr,
//            Pb = the block's rows k < m, stored) -- the peeling of
//            transform.py:513-533.
// X_u is the least-squares solution operator of the block
// A_u = 2pi sY_l(u)(theta_k), k = m..L-1, l = lo..L-1 -- square for m >= |s|,
// TALL for m < |s| (more rings than degrees).  The reference solves every
// block per call with gelsy (blocks.py:88-116); here X_u is built once per
// (plan, spin) on the device: blocks generated from the recurrence, one
// Householder QR per signed order (one CTA each), X = R^-1 Q1^T formed in
// place.  For a full-column-rank block this is the same least-squares
// solution; check=1 refuses blocks whose 1-norm condition estimate
// ||A||_1 ||X||_1 exceeds the scalar path's bound.
//
// Seeds: the reference starts each column at l = j = max(|m|, |s|) from an
// exact-rational constant (legendre.py:233-262).  osph_spin_seed computes the
// same constant on the host from the prime factorisation of the factorial
// ratio (exact exponents, 64-bit products), so it rounds like the reference's
// Fraction arithmetic.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/osph.h"
#include "plan.cuh"

#define SP_TRY(expr)                                                          \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      osph_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));     \
      return OSPH_ERR_CUDA;                                                   \
    }                                                                         \
  } while (0)

static const double kFourPi = 4.0 * OSPH_PI;  // legendre.py:26 (4.0 * math.pi)

// ---------------------------------------------------------------------------
// seed constants (host)

// Exponent of prime q in n!  (Legendre's formula).
static int64_t fact_exp(int64_t n, int64_t q) {
  int64_t e = 0;
  for (int64_t t = n / q; t > 0; t /= q) e += t;
  return e;
}

// A positive integer given by prime exponents, as mant * 2^ex with mant in [1, 2):
// odd primes multiplied into exact 64-bit chunks, each chunk rounded once into
// the 64-bit-mantissa long double (a few hundred roundings of 2^-64 at most).
struct BigVal {
  long double mant = 1.0L;
  int64_t ex = 0;
  uint64_t chunk = 1;
  void flush() {
    if (chunk == 1) return;
    int e2 = 0;
    mant = frexpl(mant * (long double)chunk, &e2) * 2.0L;
    ex += e2 - 1;
    chunk = 1;
  }
  void mul(uint64_t q, int64_t e) {
    if (q == 2) {
      ex += e;
      return;
    }
    for (int64_t i = 0; i < e; ++i) {
      if (chunk > UINT64_MAX / q) flush();
      chunk *= q;
    }
  }
};

extern "C" int osph_spin_seed(int spin, int m, int* j_out, double* scale, int* offset, int* exp_sin, int* exp_cos) {
  const int j = std::max(std::abs(m), std::abs(spin));
  if (j > 65536) {
    osph_set_error("osph_spin_seed: |m|, |spin| must be <= 65536");
    return OSPH_ERR_ARG;
  }
  if (j == 0) {
    if (j_out) *j_out = 0;
    if (scale) *scale = 1.0 / std::sqrt(kFourPi);
    if (offset) *offset = 0;
    if (exp_sin) *exp_sin = 0;
    if (exp_cos) *exp_cos = 0;
    return OSPH_OK;
  }
  // the lowest degree sits at a corner of the Wigner d-matrix: one term of the sum
  const int k = std::max(0, m - spin);
  const int esin = spin - m + 2 * k;
  const int ecos = 2 * j - esin;
  const double sign = ((k + spin) % 2 != 0) ? -1.0 : 1.0;
  // ratio2 = (j-m)! (j+m)! (j-s)! (j+s)! / [(j-s-k)! k! (s-m+k)! (j+m-k)!]^2, reduced
  const int64_t num[4] = {j - m, j + m, j - spin, j + spin};
  const int64_t den[4] = {j - spin - k, k, spin - m + k, j + m - k};
  int64_t top = 0;
  for (int64_t v : num) top = std::max(top, v);
  for (int64_t v : den) {
    if (v < 0) {
      osph_set_error("osph_spin_seed: seed degree is not at a corner of the d-matrix");
      return OSPH_ERR_ARG;
    }
    top = std::max(top, v);
  }
  std::vector<char> composite(top + 1, 0);
  BigVal N, D;
  for (int64_t q = 2; q <= top; ++q) {
    if (composite[q]) continue;
    for (int64_t r = q * q; r <= top; r += q) composite[r] = 1;
    int64_t e = 0;
    for (int64_t v : num) e += fact_exp(v, q);
    for (int64_t v : den) e -= 2 * fact_exp(v, q);
    if (e > 0) N.mul((uint64_t)q, e);
    if (e < 0) D.mul((uint64_t)q, -e);
  }
  N.flush();
  D.flush();
  // numerator.bit_length() - denominator.bit_length() of the reduced fraction, made even
  int64_t shift2 = N.ex - D.ex;
  if (shift2 & 1) shift2 -= 1;
  const long double q = (N.mant / D.mant) * ((N.ex - D.ex - shift2) ? 2.0L : 1.0L);  // ratio2 / 2^shift2
  const double base = std::sqrt((double)q);
  if (j_out) *j_out = j;
  if (scale) *scale = sign * base * std::sqrt((2 * j + 1) / kFourPi);
  if (offset) *offset = (int)(shift2 / 2);
  if (exp_sin) *exp_sin = esin;
  if (exp_cos) *exp_cos = ecos;
  return OSPH_OK;
}

// ---------------------------------------------------------------------------
// tables (device)

// Recurrence coefficients of legendre.py:296-304 for every signed order u and
// degree l in [lo, L-2]:  sY_(l+1) = ((a x - b) sY_l - c sY_(l-1)) / d, stored
// as {a/d, b/d, c/d}.  The integer parts are exact as in the reference.
__global__ void k_spin_rec(int L, int s, double4* __restrict__ rec) {
  const int u = blockIdx.y;
  const int mu = u - (L - 1);
  const int lo = max(abs(mu), abs(s));
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < L; l += gridDim.x * blockDim.x) {
    double4 r = make_double4(0.0, 0.0, 0.0, 0.0);
    if (l == 0 && lo == 0 && L > 1) r = make_double4(sqrt(3.0), 0.0, 0.0, 0.0);  // spin 0, m = 0 (legendre.py:294-295)
    if (l >= lo && l < L - 1 && l > 0) {
      const double el = (double)l, lp = el + 1.0;
      const double mm = (double)(mu * mu), ss = (double)(s * s);
      const double d = el * sqrt((lp * lp - mm) * (lp * lp - ss) / (double)(2 * l + 3));
      const double a = sqrt(2.0 * el + 1.0) * el * lp;
      const double b = sqrt(2.0 * el + 1.0) * (double)(mu * s);
      const double c = lp * sqrt((double)((int64_t)(l * l - mu * mu) * (int64_t)(l * l - s * s)) / (2.0 * el - 1.0));
      r = make_double4(a / d, b / d, c / d, 0.0);
    }
    rec[(int64_t)u * L + l] = r;
  }
}

__device__ __forceinline__ double spin_step(const double4 r, double x, double p0, double p1) {
  return fma(fma(r.x, x, -r.y), p1, -r.z * p0);
}

// Start table: per (u, ring k) the reference's seed (scale * 2^offset times
// sin(theta/2)^exp_sin cos(theta/2)^exp_cos, rescaled as legendre.py:265-270)
// and the rescaled recurrence (legendre.py:221-231) up to the first degree
// whose TRUE value ldexp(mantissa, offset) reaches 2^-500; lower degrees are
// smaller and taken as zero.  Unlike the scalar seed, the offset may start
// positive (the exact-rational scale carries 2^(shift2/2)), so the test is on
// the value, not on offset == 0.
__global__ void k_spin_start(int L, int s, const double* __restrict__ seed_scale, const int4* __restrict__ seed_int,
                             const double* __restrict__ costh, const double* __restrict__ ch,
                             const double* __restrict__ sh, const double4* __restrict__ rec, int* __restrict__ ls_tab,
                             double2* __restrict__ pstart) {
  const int u = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  const int4 si = seed_int[u];  // {lo, offset, exp_sin, exp_cos}
  double mant = seed_scale[u];
  int off = si.y;
  const double shk = sh[k], chk = ch[k];
  for (int i = 0; i < si.z; ++i) {
    mant *= shk;
    if (fabs(mant) < OSPH_TINY && mant != 0.0) {
      mant *= OSPH_UP;
      off -= 1000;
    }
  }
  for (int i = 0; i < si.w; ++i) {
    mant *= chk;
    if (fabs(mant) < OSPH_TINY && mant != 0.0) {
      mant *= OSPH_UP;
      off -= 1000;
    }
  }
  double prev = 0.0, curr = mant;
  int l = si.x;
  const double x = costh[k];
  const double4* rr = rec + (int64_t)u * L;
  // off > -1000 with |mant| <= 2^500 bounds the true value; ldexp is exact above 2^-1022
  auto in_range = [&](double v) { return off > -2000 && fabs(ldexp(v, off)) >= OSPH_TINY; };
  while (!in_range(curr) && l < L - 1) {
    const double nxt = spin_step(rr[l], x, prev, curr);
    prev = curr;
    curr = nxt;
    if (fabs(curr) > OSPH_BIG) {
      curr *= OSPH_DOWN;
      prev *= OSPH_DOWN;
      off += 1000;
    } else if (fabs(curr) < OSPH_TINY && fabs(prev) < OSPH_TINY && (curr != 0.0 || prev != 0.0)) {
      curr *= OSPH_UP;
      prev *= OSPH_UP;
      off -= 1000;
    }
    ++l;
  }
  const int64_t t = (int64_t)u * L + k;
  const bool ok = in_range(curr);
  ls_tab[t] = ok ? l : L;
  pstart[t] = ok ? make_double2(ldexp(prev, off), ldexp(curr, off)) : make_double2(0.0, 0.0);
}

// spin_table(s, mu, thetas, L) for all rings: out[(l - lo) * ld + k].
__global__ void k_spin_block(int L, int u, int lo, const double* __restrict__ costh, const double4* __restrict__ rec,
                             const int* __restrict__ ls_tab, const double2* __restrict__ pstart, double* __restrict__ out,
                             int64_t ld) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  const int64_t t = (int64_t)u * L + k;
  const int ls = ls_tab[t];
  for (int l = lo; l < min(ls, L); ++l) out[(int64_t)(l - lo) * ld + k] = 0.0;
  if (ls >= L) return;
  double p0 = pstart[t].x, p1 = pstart[t].y;
  const double x = costh[k];
  const double4* rr = rec + (int64_t)u * L;
  for (int l = ls; l < L; ++l) {
    out[(int64_t)(l - lo) * ld + k] = p1;
    if (l + 1 < L) {
      const double nxt = spin_step(rr[l], x, p0, p1);
      p0 = p1;
      p1 = nxt;
    }
  }
}

// The blocks A_u = 2pi sY_l(u)(theta_k), k = m..L-1 (rows), l = lo..L-1
// (columns), column-major into X_u's storage (the QR works in place).
__global__ void k_spin_gen(int L, int s, const int64_t* __restrict__ x_off, const double* __restrict__ costh,
                           const double4* __restrict__ rec, const int* __restrict__ ls_tab,
                           const double2* __restrict__ pstart, double* __restrict__ X) {
  const int u = blockIdx.y;
  const int mu = u - (L - 1), m = abs(mu), lo = max(m, abs(s));
  const int nr = L - m;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nr) return;
  const int k = m + i;
  double* W = X + x_off[u];
  const int64_t t = (int64_t)u * L + k;
  const int ls = ls_tab[t];
  for (int l = lo; l < min(ls, L); ++l) W[(int64_t)(l - lo) * nr + i] = 0.0;
  if (ls >= L) return;
  double p0 = pstart[t].x, p1 = pstart[t].y;
  const double x = costh[k];
  const double4* rr = rec + (int64_t)u * L;
  for (int l = ls; l < L; ++l) {
    W[(int64_t)(l - lo) * nr + i] = OSPH_TWO_PI * p1;
    if (l + 1 < L) {
      const double nxt = spin_step(rr[l], x, p0, p1);
      p0 = p1;
      p1 = nxt;
    }
  }
}

// The below-blocks Pb_u = 2pi sY_l(u)(theta_k), rings k < m (the corrections'
// operand), row-major m x (L - lo): one thread per (u, ring).
__global__ void k_spin_gen_below(int L, int s, const int64_t* __restrict__ pb_off, const double* __restrict__ costh,
                                 const double4* __restrict__ rec, const int* __restrict__ ls_tab,
                                 const double2* __restrict__ pstart, double* __restrict__ Pb) {
  const int u = blockIdx.y;
  const int mu = u - (L - 1), m = abs(mu), lo = max(m, abs(s));
  const int nc = L - lo;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  double* row = Pb + pb_off[u] + (int64_t)k * nc;
  const int64_t t = (int64_t)u * L + k;
  const int ls = ls_tab[t];
  for (int l = lo; l < min(ls, L); ++l) row[l - lo] = 0.0;
  if (ls >= L) return;
  double p0 = pstart[t].x, p1 = pstart[t].y;
  const double x = costh[k];
  const double4* rr = rec + (int64_t)u * L;
  for (int l = ls; l < L; ++l) {
    row[l - lo] = OSPH_TWO_PI * p1;
    if (l + 1 < L) {
      const double nxt = spin_step(rr[l], x, p0, p1);
      p0 = p1;
      p1 = nxt;
    }
  }
}

// ---------------------------------------------------------------------------
// per-order least-squares operators: Householder QR, one CTA per signed order

#define QR_THREADS 512

__device__ __forceinline__ double sp_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum / max (all threads get the result).
__device__ double sp_block_reduce(double v, bool is_max, double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, w) : v + w;
  }
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < QR_THREADS / 32; ++w) r = is_max ? fmax(r, red[w]) : r + red[w];
  return r;
}

// W = A_u (column-major nr x nc) -> X_u = R^-1 Q1^T (row-major nc x nr: the
// same memory, row j of X = column j of Q1).  scratch: nc*nc + nc doubles per CTA.
__global__ void __launch_bounds__(QR_THREADS) k_spin_qr(int L, int s, const int* __restrict__ orders,
                                                        const int64_t* __restrict__ x_off, double* __restrict__ X,
                                                        double* __restrict__ scratch, int64_t scratch_stride,
                                                        double* __restrict__ kappa) {
  __shared__ double red[QR_THREADS / 32];
  __shared__ double bc[2];
  const int u = orders[blockIdx.x];
  const int mu = u - (L - 1), m = abs(mu), lo = max(m, abs(s));
  const int nr = L - m, nc = L - lo;
  double* W = X + x_off[u];
  double* Rb = scratch + (int64_t)blockIdx.x * scratch_stride;
  double* tau = Rb + (int64_t)nc * nc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = QR_THREADS / 32;

  // ||A||_1 (the block as generated)
  double amax = 0.0;
  for (int c = warp; c < nc; c += NW) {
    double acc = 0.0;
    for (int r = lane; r < nr; r += 32) acc += fabs(W[(int64_t)c * nr + r]);
    amax = fmax(amax, sp_warp_sum(acc));
  }
  amax = sp_block_reduce(amax, true, red);

  // Householder QR (LAPACK dgeqr2 / dlarfg conventions)
  for (int j = 0; j < nc; ++j) {
    double* cj = W + (int64_t)j * nr;
    double ss = 0.0;
    for (int r = j + 1 + tid; r < nr; r += QR_THREADS) ss += cj[r] * cj[r];
    ss = sp_block_reduce(ss, false, red);
    if (tid == 0) {
      const double alpha = cj[j];
      double t = 0.0, vs = 0.0;
      if (ss > 0.0) {
        const double beta = -copysign(sqrt(alpha * alpha + ss), alpha);
        t = (beta - alpha) / beta;
        vs = 1.0 / (alpha - beta);
        cj[j] = beta;
      }
      tau[j] = t;
      bc[0] = vs;
      bc[1] = t;
    }
    __syncthreads();
    const double vs = bc[0], t = bc[1];
    if (t != 0.0) {
      for (int r = j + 1 + tid; r < nr; r += QR_THREADS) cj[r] *= vs;
      __syncthreads();
      for (int c = j + 1 + warp; c < nc; c += NW) {  // trailing columns: c -= t v (v . c), v = [1; cj[j+1..]]
        double* cc = W + (int64_t)c * nr;
        double w = 0.0;
        for (int r = j + 1 + lane; r < nr; r += 32) w += cj[r] * cc[r];
        const double ccj = cc[j];
        w = (sp_warp_sum(w) + ccj) * t;
        __syncwarp();
        if (lane == 0) cc[j] = ccj - w;
        for (int r = j + 1 + lane; r < nr; r += 32) cc[r] -= w * cj[r];
      }
    }
    __syncthreads();
  }
  // R (upper triangle) aside; a zero or non-finite diagonal marks the block singular
  int bad = 0;
  for (int idx = tid; idx < nc * nc; idx += QR_THREADS) {
    const int a = idx / nc, b = idx - a * nc;
    const double v = b >= a ? W[(int64_t)b * nr + a] : 0.0;
    Rb[idx] = v;
    if (a == b && !(fabs(v) > 0.0 && fabs(v) <= 1.0e300)) bad = 1;
  }
  bad = __syncthreads_or(bad);
  // Q1 = H_0 ... H_(nc-1) [I; 0] in place (LAPACK dorg2r)
  for (int i = nc - 1; i >= 0; --i) {
    double* ci = W + (int64_t)i * nr;
    const double t = tau[i];
    if (i < nc - 1 && t != 0.0) {
      for (int c = i + 1 + warp; c < nc; c += NW) {
        double* cc = W + (int64_t)c * nr;
        double w = 0.0;
        for (int r = i + 1 + lane; r < nr; r += 32) w += ci[r] * cc[r];
        const double cci = cc[i];
        w = (sp_warp_sum(w) + cci) * t;
        __syncwarp();
        if (lane == 0) cc[i] = cci - w;
        for (int r = i + 1 + lane; r < nr; r += 32) cc[r] -= w * ci[r];
      }
      __syncthreads();
    }
    for (int r = tid; r < nr; r += QR_THREADS) ci[r] = r > i ? -t * ci[r] : (r == i ? 1.0 - t : 0.0);
    __syncthreads();
  }
  // X = R^-1 Q1^T: column i of X (elements W[j*nr + i]) by back substitution, one thread per i
  double xmax = 0.0;
  if (!bad) {
    for (int i = tid; i < nr; i += QR_THREADS) {
      double colsum = 0.0;
      for (int j = nc - 1; j >= 0; --j) {
        const double* rj = Rb + (int64_t)j * nc;
        double acc = W[(int64_t)j * nr + i];
        for (int t2 = j + 1; t2 < nc; ++t2) acc = fma(-rj[t2], W[(int64_t)t2 * nr + i], acc);
        const double v = acc / rj[j];
        W[(int64_t)j * nr + i] = v;
        colsum += fabs(v);
      }
      if (!(colsum <= 1.0e300)) bad = 1;
      xmax = fmax(xmax, colsum);
    }
  }
  bad = __syncthreads_or(bad);
  xmax = sp_block_reduce(xmax, true, red);
  if (bad)  // a singular block solves to zero (check=1 refuses it first)
    for (int64_t idx = tid; idx < (int64_t)nr * nc; idx += QR_THREADS) W[idx] = 0.0;
  if (tid == 0) kappa[u] = bad ? INFINITY : amax * xmax;
}

// ---------------------------------------------------------------------------
// per-call kernels

#define SOLVE_MB 4

// x_(+-m) = X_(+-m) g_(+-m) for maps [b0, b0 + SOLVE_MB): one warp per row (degree
// lo + j), lanes over the rings; writes flm and the order's x to xbuf.
__global__ void __launch_bounds__(256) k_spin_solve(int L, int s, int m, int B, const double* __restrict__ X,
                                                    const int64_t* __restrict__ x_off, const double2* __restrict__ R,
                                                    double2* __restrict__ xbuf, double2* __restrict__ flm) {
  pdl_start();
  const int sg = blockIdx.y;  // 0: +m, 1: -m
  const int mu = sg ? -m : m, u = mu + L - 1;
  const int lo = max(m, abs(s)), nr = L - m, nc = L - lo;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= nc) return;
  const double* Xr = X + x_off[u] + (int64_t)j * nr;
  const int64_t npos = (int64_t)L * (L + 1) / 2, p0 = packed_pos(L, m, 0);
  const int b0 = blockIdx.z * SOLVE_MB;
  double ar[SOLVE_MB], ai[SOLVE_MB];
#pragma unroll
  for (int q = 0; q < SOLVE_MB; ++q) ar[q] = ai[q] = 0.0;
  for (int i = lane; i < nr; i += 32) {
    const double xv = __ldg(Xr + i);
#pragma unroll
    for (int q = 0; q < SOLVE_MB; ++q) {
      if (b0 + q < B) {
        const double2 g = R[((int64_t)(b0 + q) * npos + p0 + i) * 2 + sg];
        ar[q] = fma(xv, g.x, ar[q]);
        ai[q] = fma(xv, g.y, ai[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < SOLVE_MB; ++q) {
    const double vr = sp_warp_sum(ar[q]), vi = sp_warp_sum(ai[q]);
    if (lane == 0 && b0 + q < B) {
      const int64_t l = lo + j;
      const double2 v = make_double2(vr, vi);
      xbuf[((int64_t)(b0 + q) * 2 + sg) * L + j] = v;
      flm[(int64_t)(b0 + q) * L * L + l * l + l + mu] = v;
    }
  }
}

// Corrections of order m on the rings k < m (transform.py:527-532 through the
// spectra): G_(+-m)(theta_k) = Pb_(+-m)[k, :] x_(+-m), subtracted from the bins
// the tones e^(+-i m phi) alias to on ring k.  One warp per ring (lanes over
// the degrees: coalesced Pb rows) and chunk of 4 maps; lane 0 writes both
// tones of a map: single writer per bin (deterministic).
#define CORR_MB 4
__global__ void __launch_bounds__(256) k_spin_corr(int L, int s, int m, int B, const double* __restrict__ Pb,
                                                   const int64_t* __restrict__ pb_off,
                                                   const double2* __restrict__ xbuf, double2* __restrict__ R) {
  pdl_start();
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= m) return;
  const int lo = max(m, abs(s)), nc = L - lo;
  const double* rp = Pb + pb_off[m + L - 1] + (int64_t)k * nc;
  const double* rn = Pb + pb_off[-m + L - 1] + (int64_t)k * nc;
  const int64_t npos = (int64_t)L * (L + 1) / 2;
  const int nk = 2 * k + 1, rr = m % nk;
  const int tm = rr == 0 ? 0 : (rr <= k ? rr : nk - rr);
  const int slot_p = rr <= k ? 0 : 1;  // +m -> bin rr: (rr, +) if rr <= k else (nk - rr, -); -m the other slot
  {
    const int b0 = blockIdx.y * CORR_MB;
    double a[CORR_MB][4];
#pragma unroll
    for (int q = 0; q < CORR_MB; ++q) a[q][0] = a[q][1] = a[q][2] = a[q][3] = 0.0;
    for (int l = lane; l < nc; l += 32) {
      const double pp = __ldg(rp + l), pn = __ldg(rn + l);
#pragma unroll
      for (int q = 0; q < CORR_MB; ++q) {
        if (b0 + q < B) {
          const double2 xp = xbuf[((int64_t)(b0 + q) * 2 + 0) * L + l];
          const double2 xn = xbuf[((int64_t)(b0 + q) * 2 + 1) * L + l];
          a[q][0] = fma(pp, xp.x, a[q][0]);
          a[q][1] = fma(pp, xp.y, a[q][1]);
          a[q][2] = fma(pn, xn.x, a[q][2]);
          a[q][3] = fma(pn, xn.y, a[q][3]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < CORR_MB; ++q) {
      const double vpr = sp_warp_sum(a[q][0]), vpi = sp_warp_sum(a[q][1]);
      const double vnr = sp_warp_sum(a[q][2]), vni = sp_warp_sum(a[q][3]);
      if (lane == 0 && b0 + q < B) {
        double2* e = R + ((int64_t)(b0 + q) * npos + packed_pos(L, tm, k - tm)) * 2;
        if (rr == 0) {  // both tones land in bin 0 (stored at (0, k), + slot)
          e->x -= vpr + vnr;
          e->y -= vpi + vni;
        } else {
          e[slot_p].x -= vpr;
          e[slot_p].y -= vpi;
          e[1 - slot_p].x -= vnr;
          e[1 - slot_p].y -= vni;
        }
      }
    }
  }
}

// G_(+-m)(theta_k) = sum_l sY_l(+-m)(theta_k) f_l(+-m) in the ring kernels' layout
// [m][k][4B] (cols 4b + {0,1}: +m, {2,3}: -m times (-1)^m, which fold_bin undoes;
// 2pi is applied by the ring kernels).  One thread per (ring, order), 4 maps.
__global__ void __launch_bounds__(128) k_spin_synth(int L, int s, int B, const double* __restrict__ costh,
                                                    const double4* __restrict__ rec, const int* __restrict__ ls_tab,
                                                    const double2* __restrict__ pstart,
                                                    const double2* __restrict__ flm, double* __restrict__ G) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  const int b0 = blockIdx.z * 4;
  if (k >= L) return;
  const double x = costh[k];
  for (int sg = 0; sg < 2; ++sg) {
    double ar[4] = {0.0, 0.0, 0.0, 0.0}, ai[4] = {0.0, 0.0, 0.0, 0.0};
    const int mu = sg ? -m : m, u = mu + L - 1;
    const int64_t t = (int64_t)u * L + k;
    const int ls = (sg && m == 0) ? L : ls_tab[t];
    if (ls < L) {
      double p0 = pstart[t].x, p1 = pstart[t].y;
      const double4* rr = rec + (int64_t)u * L;
      for (int l = ls; l < L; ++l) {
        const int64_t idx = (int64_t)l * l + l + mu;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (b0 + q < B) {
            const double2 f = __ldg(flm + (int64_t)(b0 + q) * L * L + idx);
            ar[q] = fma(p1, f.x, ar[q]);
            ai[q] = fma(p1, f.y, ai[q]);
          }
        }
        if (l + 1 < L) {
          const double nxt = spin_step(rr[l], x, p0, p1);
          p0 = p1;
          p1 = nxt;
        }
      }
    }
    const double sgn = (sg && (m & 1)) ? -1.0 : 1.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (b0 + q < B) {
        double* g = G + ((int64_t)m * L + k) * 4 * B + 4 * (b0 + q) + 2 * sg;
        g[0] = sgn * ar[q];
        g[1] = sgn * ai[q];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host side

static void spin_state_free(SpinState* st) {
  if (!st) return;
  void* ptrs[] = {st->d_ls, st->d_pstart, st->d_rec, st->d_x, st->d_x_off, st->d_pb, st->d_pb_off, st->d_kappa};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  delete st;
}

void spin_free(osph_plan* p) {
  for (SpinState* st : p->spins) spin_state_free(st);
  p->spins.clear();
  if (p->d_spin_xbuf) cudaFree(p->d_spin_xbuf);
  p->d_spin_xbuf = nullptr;
}

static int check_spin(const osph_plan* p, int spin) {
  if (!p) {
    osph_set_error("plan is NULL");
    return OSPH_ERR_ARG;
  }
  if (std::abs(spin) >= p->L) {  // transform.py:482-483, 510-511
    osph_set_error("spin " + std::to_string(spin) + " invalid for band limit " + std::to_string(p->L));
    return OSPH_ERR_ORDER;
  }
  if (!p->group_devs.empty() || p->shard_mode) {
    osph_set_error("spin transforms run on single-device, unsharded plans");
    return OSPH_ERR_ARG;
  }
  return OSPH_OK;
}

// Tables of spin s (the plan keeps the two most recently used spins).
static int spin_tables(osph_plan* p, int s, SpinState** out) {
  for (size_t i = 0; i < p->spins.size(); ++i) {
    if (p->spins[i]->s == s) {
      SpinState* st = p->spins[i];
      p->spins.erase(p->spins.begin() + i);
      p->spins.insert(p->spins.begin(), st);  // most recent first
      *out = st;
      return OSPH_OK;
    }
  }
  while (p->spins.size() >= 2) {
    SP_TRY(cudaStreamSynchronize(p->stream));
    spin_state_free(p->spins.back());
    p->spins.pop_back();
  }
  const int L = p->L, U = 2 * L - 1;
  cudaStream_t strm = p->stream;
  std::vector<double> scale(U);
  std::vector<int4> seeds(U);
  for (int u = 0; u < U; ++u) {
    const int mu = u - (L - 1);
    int j = 0, off = 0, es = 0, ec = 0;
    int rc = osph_spin_seed(s, mu, &j, &scale[u], &off, &es, &ec);
    if (rc) return rc;
    seeds[u] = make_int4(j, off, es, ec);
  }
  std::vector<double> ch(L), sh(L);
  for (int k = 0; k < L; ++k) {  // np.cos(thetas / 2.0), np.sin(thetas / 2.0) (legendre.py:263-264)
    ch[k] = std::cos(p->h_thetas[k] / 2.0);
    sh[k] = std::sin(p->h_thetas[k] / 2.0);
  }
  SpinState* st = new SpinState();
  st->s = s;
  double *d_scale = nullptr, *d_ch = nullptr, *d_sh = nullptr;
  int4* d_seeds = nullptr;
  auto fail = [&](cudaError_t e) {
    osph_set_error(std::string("spin tables: ") + cudaGetErrorString(e));
    cudaFree(d_scale);
    cudaFree(d_ch);
    cudaFree(d_sh);
    cudaFree(d_seeds);
    spin_state_free(st);
    return OSPH_ERR_CUDA;
  };
  cudaError_t e;
  const size_t nt = (size_t)U * L;
  if ((e = cudaMalloc(&st->d_ls, sizeof(int) * nt)) || (e = cudaMalloc(&st->d_pstart, sizeof(double2) * nt)) ||
      (e = cudaMalloc(&st->d_rec, sizeof(double4) * nt)) || (e = cudaMalloc(&d_scale, sizeof(double) * U)) ||
      (e = cudaMalloc(&d_seeds, sizeof(int4) * U)) || (e = cudaMalloc(&d_ch, sizeof(double) * L)) ||
      (e = cudaMalloc(&d_sh, sizeof(double) * L)))
    return fail(e);
  if ((e = cudaMemcpyAsync(d_scale, scale.data(), sizeof(double) * U, cudaMemcpyHostToDevice, strm)) ||
      (e = cudaMemcpyAsync(d_seeds, seeds.data(), sizeof(int4) * U, cudaMemcpyHostToDevice, strm)) ||
      (e = cudaMemcpyAsync(d_ch, ch.data(), sizeof(double) * L, cudaMemcpyHostToDevice, strm)) ||
      (e = cudaMemcpyAsync(d_sh, sh.data(), sizeof(double) * L, cudaMemcpyHostToDevice, strm)))
    return fail(e);
  k_spin_rec<<<dim3((L + 127) / 128, U), 128, 0, strm>>>(L, s, st->d_rec);
  k_spin_start<<<dim3((L + 127) / 128, U), 128, 0, strm>>>(L, s, d_scale, d_seeds, p->d_cos, d_ch, d_sh, st->d_rec,
                                                           st->d_ls, st->d_pstart);
  if ((e = cudaGetLastError()) || (e = cudaStreamSynchronize(strm))) return fail(e);
  cudaFree(d_scale);
  cudaFree(d_ch);
  cudaFree(d_sh);
  cudaFree(d_seeds);
  p->spins.insert(p->spins.begin(), st);
  *out = st;
  return OSPH_OK;
}

// The least-squares operators X_u of every signed order (once per plan and spin).
static int spin_factor(osph_plan* p, SpinState* st) {
  if (st->factored) {
    st->factor_seconds = 0.0;
    return OSPH_OK;
  }
  const int L = p->L, U = 2 * L - 1, s = st->s, as = std::abs(s);
  cudaStream_t strm = p->stream;
  st->h_x_off.assign(U + 1, 0);
  for (int u = 0; u < U; ++u) {
    const int m = std::abs(u - (L - 1)), lo = std::max(m, as);
    st->h_x_off[u + 1] = st->h_x_off[u] + (int64_t)(L - lo) * (L - m);
  }
  st->h_pb_off.assign(U + 1, 0);
  for (int u = 0; u < U; ++u) {
    const int m = std::abs(u - (L - 1)), lo = std::max(m, as);
    st->h_pb_off[u + 1] = st->h_pb_off[u] + (int64_t)m * (L - lo);
  }
  SP_TRY(cudaMalloc(&st->d_x, sizeof(double) * std::max<int64_t>(1, st->h_x_off[U])));
  SP_TRY(cudaMalloc(&st->d_x_off, sizeof(int64_t) * (U + 1)));
  SP_TRY(cudaMalloc(&st->d_pb, sizeof(double) * std::max<int64_t>(1, st->h_pb_off[U])));
  SP_TRY(cudaMalloc(&st->d_pb_off, sizeof(int64_t) * (U + 1)));
  SP_TRY(cudaMemcpyAsync(st->d_pb_off, st->h_pb_off.data(), sizeof(int64_t) * (U + 1), cudaMemcpyHostToDevice,
                         strm));
  SP_TRY(cudaMalloc(&st->d_kappa, sizeof(double) * U));
  SP_TRY(cudaMemcpyAsync(st->d_x_off, st->h_x_off.data(), sizeof(int64_t) * (U + 1), cudaMemcpyHostToDevice, strm));
  cudaEvent_t e0, e1;
  SP_TRY(cudaEventCreate(&e0));
  SP_TRY(cudaEventCreate(&e1));
  SP_TRY(cudaEventRecord(e0, strm));
  k_spin_gen<<<dim3((L + 127) / 128, U), 128, 0, strm>>>(L, s, st->d_x_off, p->d_cos, st->d_rec, st->d_ls,
                                                         st->d_pstart, st->d_x);
  k_spin_gen_below<<<dim3((L + 127) / 128, U), 128, 0, strm>>>(L, s, st->d_pb_off, p->d_cos, st->d_rec, st->d_ls,
                                                               st->d_pstart, st->d_pb);
  SP_TRY(cudaGetLastError());
  // largest blocks first; waves of CTAs sized so the R scratch stays bounded
  std::vector<int> order(U);
  for (int u = 0; u < U; ++u) order[u] = u;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return std::abs(a - (L - 1)) < std::abs(b - (L - 1));
  });
  int sms = 0;
  SP_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device));
  const int ncmax = L - as;
  const int64_t stride = (int64_t)ncmax * ncmax + ncmax + 1;
  const int64_t budget = (int64_t)1 << 28;  // doubles of R scratch (2 GiB)
  const int wave = (int)std::max<int64_t>(1, std::min<int64_t>(U, std::min<int64_t>(4 * (int64_t)sms, budget / stride)));
  int* d_orders = nullptr;
  double* d_scr = nullptr;
  SP_TRY(cudaMalloc(&d_orders, sizeof(int) * U));
  SP_TRY(cudaMalloc(&d_scr, sizeof(double) * stride * wave));
  SP_TRY(cudaMemcpyAsync(d_orders, order.data(), sizeof(int) * U, cudaMemcpyHostToDevice, strm));
  for (int w0 = 0; w0 < U; w0 += wave) {
    const int cnt = std::min(wave, U - w0);
    k_spin_qr<<<cnt, QR_THREADS, 0, strm>>>(L, s, d_orders + w0, st->d_x_off, st->d_x, d_scr, stride, st->d_kappa);
    SP_TRY(cudaGetLastError());
  }
  SP_TRY(cudaEventRecord(e1, strm));
  st->h_kappa.assign(U, 0.0);
  SP_TRY(cudaMemcpyAsync(st->h_kappa.data(), st->d_kappa, sizeof(double) * U, cudaMemcpyDeviceToHost, strm));
  SP_TRY(cudaStreamSynchronize(strm));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  st->factor_seconds = ms * 1e-3;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d_orders);
  cudaFree(d_scr);
  st->factored = true;
  return OSPH_OK;
}

static int check_io(osph_plan* p, int B, const void* a, void* b, int kind) {
  if (B < 1 || B > p->max_batch) {
    osph_set_error("batch " + std::to_string(B) + " outside [1, max_batch=" + std::to_string(p->max_batch) + "]");
    return OSPH_ERR_ARG;
  }
  if (!a || !b) {
    osph_set_error("NULL data pointer");
    return OSPH_ERR_ARG;
  }
  if (kind & ~(OSPH_DEVICE | OSPH_ASYNC)) {
    osph_set_error("spin transforms take OSPH_HOST / OSPH_DEVICE (| OSPH_ASYNC) pointers");
    return OSPH_ERR_ARG;
  }
  if ((kind & OSPH_ASYNC) && !(kind & OSPH_DEVICE)) {
    osph_set_error("OSPH_ASYNC requires OSPH_DEVICE pointers");
    return OSPH_ERR_ARG;
  }
  if (!p->dft_ok) {
    osph_set_error("ring DFT length exceeds the two-CTA Bluestein FFT (transforms need L <= 4096)");
    return OSPH_ERR_ARG;
  }
  return OSPH_OK;
}

extern "C" int osph_spin_block(osph_plan* p, int spin, int m, double* out, int64_t ld, int kind) {
  DeviceGuard guard;
  osph_set_error("");
  if (!p || !out) {
    osph_set_error("NULL plan or output pointer");
    return OSPH_ERR_ARG;
  }
  const int L = p->L;
  const int lo = std::max(std::abs(m), std::abs(spin));
  if (lo >= L) {  // legendre.py:285-288
    osph_set_error("order " + std::to_string(m) + ", spin " + std::to_string(spin) + " invalid for band limit " +
                   std::to_string(L));
    return OSPH_ERR_ORDER;
  }
  if (!p->group_devs.empty()) {
    osph_set_error("spin tables need a single-device plan");
    return OSPH_ERR_ARG;
  }
  if (ld < L || !(kind & OSPH_DEVICE) || (kind & ~(OSPH_DEVICE | OSPH_ASYNC))) {
    osph_set_error("osph_spin_block needs a device pointer and ld >= L");
    return OSPH_ERR_ARG;
  }
  SP_TRY(cudaSetDevice(p->device));
  SpinState* st = nullptr;
  int rc = spin_tables(p, spin, &st);
  if (rc) return rc;
  k_spin_block<<<(L + 127) / 128, 128, 0, p->stream>>>(L, m + L - 1, lo, p->d_cos, st->d_rec, st->d_ls, st->d_pstart,
                                                       out, ld);
  SP_TRY(cudaGetLastError());
  if (!(kind & OSPH_ASYNC)) SP_TRY(cudaStreamSynchronize(p->stream));
  return OSPH_OK;
}

extern "C" int osph_spin_inverse(osph_plan* p, int spin, int B, const void* flm, void* samples, int kind) {
  DeviceGuard guard;
  osph_set_error("");
  int rc = check_spin(p, spin);
  if (rc) return rc;
  if (spin == 0) return osph_inverse(p, B, flm, samples, kind);  // the scalar path, bit for bit (transform.py:484-485)
  if ((rc = check_io(p, B, flm, samples, kind))) return rc;
  SP_TRY(cudaSetDevice(p->device));
  if ((rc = ensure_inverse(p))) return rc;
  const bool host = !(kind & OSPH_DEVICE);
  if (host && (rc = ensure_io(p))) return rc;
  SpinState* st = nullptr;
  if ((rc = spin_tables(p, spin, &st))) return rc;
  const int L = p->L;
  const size_t bytes = sizeof(double2) * (size_t)B * L * L;
  cudaStream_t strm = p->stream;
  p->launches = 0;
  const double2* src = (const double2*)flm;
  double2* dst = host ? p->d_out : (double2*)samples;
  if (host) {
    SP_TRY(cudaMemcpyAsync(p->d_in, flm, bytes, cudaMemcpyHostToDevice, strm));
    src = p->d_in;
  }
  SP_TRY(cudaEventRecord(p->ev[0], strm));
  SP_TRY(cudaEventRecord(p->ev[1], strm));
  k_spin_synth<<<dim3((L + 127) / 128, L, (B + 3) / 4), 128, 0, strm>>>(L, spin, B, p->d_cos, st->d_rec, st->d_ls,
                                                                        st->d_pstart, src, p->d_g);
  SP_TRY(cudaGetLastError());
  p->launches++;
  SP_TRY(cudaEventRecord(p->ev[2], strm));
  SP_TRY(launch_ring_inverse(p, B, dst));
  SP_TRY(cudaEventRecord(p->ev[3], strm));
  if (host) SP_TRY(cudaMemcpyAsync(samples, p->d_out, bytes, cudaMemcpyDeviceToHost, strm));
  p->have_inv = true;
  if (!(kind & OSPH_ASYNC)) SP_TRY(cudaStreamSynchronize(strm));
  return OSPH_OK;
}

extern "C" int osph_spin_forward(osph_plan* p, int spin, int B, const void* samples, void* flm, int kind, int check,
                                 osph_stats* stats) {
  DeviceGuard guard;
  osph_set_error("");
  int rc = check_spin(p, spin);
  if (rc) return rc;
  if (spin == 0) return osph_forward(p, B, samples, flm, kind, check, stats);  // transform.py:512-513
  if ((rc = check_io(p, B, samples, flm, kind))) return rc;
  if ((kind & OSPH_ASYNC) && check) {
    osph_set_error("check=1 needs a host-blocking call (drop OSPH_ASYNC or pass check=0)");
    return OSPH_ERR_ARG;
  }
  SP_TRY(cudaSetDevice(p->device));
  const bool host = !(kind & OSPH_DEVICE);
  if (host && (rc = ensure_io(p))) return rc;
  if ((rc = ensure_spectra(p))) return rc;
  const int L = p->L, U = 2 * L - 1;
  if (!p->d_spin_xbuf) SP_TRY(cudaMalloc(&p->d_spin_xbuf, sizeof(double2) * 2 * L * (size_t)p->max_batch));
  SpinState* st = nullptr;
  if ((rc = spin_tables(p, spin, &st))) return rc;
  if ((rc = spin_factor(p, st))) return rc;
  if (check) {  // the reference raises at the first failing solve of its sweep: m descending, +m before -m
    for (int m = L - 1; m >= 0; --m) {
      for (int sg = 0; sg < (m ? 2 : 1); ++sg) {
        const int mu = sg ? -m : m;
        const double kap = st->h_kappa[mu + L - 1];
        if (!(kap <= 2.0e14)) {
          if (stats) {
            stats->failed_order = mu;
            stats->failed_kappa = kap;
          }
          char buf[160];
          snprintf(buf, sizeof buf, "order %d system is numerically singular (condition number %.3e)", mu, kap);
          osph_set_error(buf);
          return OSPH_ERR_ILLCOND;
        }
      }
    }
  }
  (void)U;
  const size_t bytes = sizeof(double2) * (size_t)B * L * L;
  cudaStream_t strm = p->stream;
  p->launches = 0;
  const double2* src = (const double2*)samples;
  double2* out = host ? p->d_out : (double2*)flm;
  if (host) {
    SP_TRY(cudaMemcpyAsync(p->d_in, samples, bytes, cudaMemcpyHostToDevice, strm));
    src = p->d_in;
  }
  SP_TRY(cudaMemsetAsync(out, 0, bytes, strm));  // degrees below |spin| come back zero (transform.py:507)
  SP_TRY(cudaEventRecord(p->ev[4], strm));
  SP_TRY(launch_ring_forward(p, B, src, 0, -1, /*plain=*/true));
  SP_TRY(cudaEventRecord(p->ev[5], strm));
  SP_TRY(cudaEventRecord(p->ev[6], strm));
  SP_TRY(cudaEventRecord(p->ev[7], strm));
  SP_TRY(cudaEventRecord(p->ev[8], strm));
  for (int m = L - 1; m >= 0; --m) {
    const int lo = std::max(m, std::abs(spin)), nc = L - lo;
    SP_TRY(launch_pdl(k_spin_solve, dim3((nc + 7) / 8, m ? 2 : 1, (B + SOLVE_MB - 1) / SOLVE_MB), dim3(256), 0, strm,
                      L, spin, m, B, (const double*)st->d_x, (const int64_t*)st->d_x_off, (const double2*)p->d_r,
                      p->d_spin_xbuf, out));
    p->launches++;
    if (m > 0) {
      SP_TRY(launch_pdl(k_spin_corr, dim3((m + 7) / 8, (B + CORR_MB - 1) / CORR_MB), dim3(256), 0, strm, L, spin, m, B, (const double*)st->d_pb,
                        (const int64_t*)st->d_pb_off, (const double2*)p->d_spin_xbuf, p->d_r));
      p->launches++;
    }
  }
  SP_TRY(cudaEventRecord(p->ev[9], strm));
  if (host) SP_TRY(cudaMemcpyAsync(flm, p->d_out, bytes, cudaMemcpyDeviceToHost, strm));
  p->have_fwd = true;
  if (kind & OSPH_ASYNC) return OSPH_OK;
  SP_TRY(cudaStreamSynchronize(strm));
  if (stats) {
    float t_ring = 0, t_sweep = 0;
    cudaEventElapsedTime(&t_ring, p->ev[4], p->ev[5]);
    cudaEventElapsedTime(&t_sweep, p->ev[8], p->ev[9]);
    stats->factor_seconds = st->factor_seconds;
    stats->sweep_seconds = t_sweep * 1e-3;
    stats->solve_seconds = st->factor_seconds + t_sweep * 1e-3;
    stats->total_seconds = (t_ring + t_sweep) * 1e-3 + st->factor_seconds;
    stats->orders = L;
    stats->failed_order = -1;
    stats->failed_kappa = 0.0;
  }
  return OSPH_OK;
}
