/*
 * oracle_kernels.c -- CPU restatement of the reference (optisph) hot-path
 * inner loops, in plain C.  TEST INFRASTRUCTURE ONLY: this file is the
 * checker for the CUDA path (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline / --impl reference legs).  The product never links it.
 *
 * Each function restates one numba kernel of the reference; the loop order
 * and floating-point operation order follow the cited lines so results agree
 * with the reference to the last few ulps (validated in tests/test_oracle.py
 * against fixtures produced by the reference itself).
 *
 *   oracle_legendre_table  <- pkg/src/optisph/legendre.py:64-96 (_legendre_kernel)
 *                             and 110-143 (legendre_table seed/sign logic)
 *   oracle_g_accumulate    <- pkg/src/optisph/transform.py:143-201 (_g_accumulate)
 *   oracle_fold_bins       <- pkg/src/optisph/transform.py:204-218 (_fold_bins)
 *   oracle_peel_analyze    <- pkg/src/optisph/transform.py:221-242 (_peel_analyze)
 *   oracle_peel_update     <- pkg/src/optisph/transform.py:245-261 (_peel_update)
 */
#include <math.h>
#include <stdint.h>
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#include <stdint.h>

#define OR_BIG 0x1p500
#define OR_TINY 0x1p-500
#define OR_UP 0x1p1000
#define OR_DOWN 0x1p-1000

/* Rescaled upward recurrence for one order over many co-latitudes.
 * out is row-major [nth][ncols]; seed0, seed_fac, a_curr, a_next as in
 * legendre.py:134-137 / 99-107. */
void oracle_legendre_kernel(const double* costh, const double* sinth, int64_t nth, int64_t am,
                            int64_t ncols, double seed0, const double* seed_fac,
                            const double* a_curr, const double* a_next, double* out) {
  for (int64_t i = 0; i < nth; ++i) {
    const double c = costh[i], s = sinth[i];
    double mant = seed0;
    int64_t off = 0;
    for (int64_t q = 0; q < am; ++q) {
      mant *= s * seed_fac[q];
      if (-OR_TINY < mant && mant < OR_TINY && mant != 0.0) {
        mant *= OR_UP;
        off -= 1000;
      }
    }
    double* row = out + i * ncols;
    row[0] = ldexp(mant, (int)off);
    double prev = 0.0, curr = mant;
    for (int64_t j = 0; j < ncols - 1; ++j) {
      double nxt = (c * curr - a_curr[j] * prev) / a_next[j];
      prev = curr;
      curr = nxt;
      double ac = fabs(curr);
      if (ac > OR_BIG) {
        curr *= OR_DOWN;
        prev *= OR_DOWN;
        off += 1000;
      } else if (ac < OR_TINY && fabs(prev) < OR_TINY && (curr != 0.0 || prev != 0.0)) {
        curr *= OR_UP;
        prev *= OR_UP;
        off -= 1000;
      }
      row[j + 1] = ldexp(curr, (int)off);
    }
  }
}

/* Fused synthesis: out[i][m][0..3] = sum_l P_lm(theta_i) * fcols[idx][0..3]
 * (transform.py:143-201).  fcols is [L(L+1)/2][4], out is [nth][L][4]. */
void oracle_g_accumulate(const double* costh, const double* sinth, int64_t nth,
                         const double* fcols, const double* seed_fac, const double* a_curr,
                         const double* a_next, const int64_t* offsets, int64_t L, double* out) {
  const double four_pi = 4.0 * M_PI;
  for (int64_t i = 0; i < nth; ++i) {
    const double c = costh[i], s = sinth[i];
    for (int64_t m = 0; m < L; ++m) {
      const int64_t base = offsets[m];
      double mant = sqrt((double)(2 * m + 1) / four_pi);
      if (m % 2) mant = -mant;
      int64_t off = 0;
      for (int64_t q = 0; q < m; ++q) {
        mant *= s * seed_fac[q];
        if (-OR_TINY < mant && mant < OR_TINY && mant != 0.0) {
          mant *= OR_UP;
          off -= 1000;
        }
      }
      double prev = 0.0, curr = mant;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      const int64_t ncols = L - m;
      for (int64_t j = 0; j < ncols; ++j) {
        const double v = ldexp(curr, (int)off);
        const int64_t idx = base + j;
        a0 += v * fcols[4 * idx + 0];
        a1 += v * fcols[4 * idx + 1];
        a2 += v * fcols[4 * idx + 2];
        a3 += v * fcols[4 * idx + 3];
        if (j < ncols - 1) {
          double nxt = (c * curr - a_curr[idx] * prev) / a_next[idx];
          prev = curr;
          curr = nxt;
          double ac = fabs(curr);
          if (ac > OR_BIG) {
            curr *= OR_DOWN;
            prev *= OR_DOWN;
            off += 1000;
          } else if (ac < OR_TINY && fabs(prev) < OR_TINY && (curr != 0.0 || prev != 0.0)) {
            curr *= OR_UP;
            prev *= OR_UP;
            off -= 1000;
          }
        }
      }
      double* o = out + (i * L + m) * 4;
      o[0] = a0;
      o[1] = a1;
      o[2] = a2;
      o[3] = a3;
    }
  }
}

/* Tone folding (transform.py:204-218).  g_plus/g_minus are complex [L][L]
 * stored as interleaved (re, im); bins complex [L*L]. */
void oracle_fold_bins(const double* g_plus, const double* g_minus, int64_t L, double* bins) {
  for (int64_t k = 0; k < L; ++k) {
    const int64_t n = 2 * k + 1, s = k * k;
    int64_t mp = 0;
    for (int64_t m = 0; m < L; ++m) {
      bins[2 * (s + mp)] += g_plus[2 * (k * L + m)];
      bins[2 * (s + mp) + 1] += g_plus[2 * (k * L + m) + 1];
      if (m > 0) {
        const int64_t mn = mp != 0 ? n - mp : 0;
        bins[2 * (s + mn)] += g_minus[2 * (k * L + m)];
        bins[2 * (s + mn) + 1] += g_minus[2 * (k * L + m) + 1];
      }
      if (++mp == n) mp = 0;
    }
  }
}

/* Exact two-bin ring DFT for rings k >= m (transform.py:221-242).
 * buf, roots complex [L*L]; out_p/out_n complex [L-m]. */
void oracle_peel_analyze(const double* buf, const double* roots, int64_t m, int64_t L,
                         double* out_p, double* out_n) {
  const double two_pi = 2.0 * M_PI;
  for (int64_t k = m; k < L; ++k) {
    const int64_t n = 2 * k + 1, s = k * k, step = m % n;
    double pr = 0.0, pi = 0.0, nr = 0.0, ni = 0.0;
    int64_t mj = 0;
    for (int64_t j = 0; j < n; ++j) {
      const double tr = roots[2 * (s + mj)], ti = roots[2 * (s + mj) + 1];
      const double vr = buf[2 * (s + j)], vi = buf[2 * (s + j) + 1];
      /* acc_p += v * conj(t); acc_n += v * t */
      pr += vr * tr + vi * ti;
      pi += vi * tr - vr * ti;
      nr += vr * tr - vi * ti;
      ni += vi * tr + vr * ti;
      mj += step;
      if (mj >= n) mj -= n;
    }
    const double delta = two_pi / (double)n;
    out_p[2 * (k - m)] = delta * pr;
    out_p[2 * (k - m) + 1] = delta * pi;
    out_n[2 * (k - m)] = delta * nr;
    out_n[2 * (k - m) + 1] = delta * ni;
  }
}

/* Spatial-domain subtraction of the order +-m contribution from rings k < m
 * (transform.py:245-261).  big_gp/big_gn complex [nk]. */
void oracle_peel_update(double* buf, const double* roots, int64_t m, int64_t nk,
                        const double* big_gp, const double* big_gn) {
  const double two_pi = 2.0 * M_PI;
  for (int64_t k = 0; k < nk; ++k) {
    const int64_t n = 2 * k + 1, s = k * k, step = m % n;
    const double cpr = big_gp[2 * k] / two_pi, cpi = big_gp[2 * k + 1] / two_pi;
    const double cnr = big_gn[2 * k] / two_pi, cni = big_gn[2 * k + 1] / two_pi;
    int64_t mj = 0;
    for (int64_t j = 0; j < n; ++j) {
      const double tr = roots[2 * (s + mj)], ti = roots[2 * (s + mj) + 1];
      /* buf -= cp * t + cn * conj(t) */
      const double ur = (cpr * tr - cpi * ti) + (cnr * tr + cni * ti);
      const double ui = (cpr * ti + cpi * tr) + (cni * tr - cnr * ti);
      buf[2 * (s + j)] -= ur;
      buf[2 * (s + j) + 1] -= ui;
      mj += step;
      if (mj >= n) mj -= n;
    }
  }
}
