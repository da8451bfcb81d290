// pivots.cu -- the grid's pivot order for every per-order block, once per plan.
//
// The per-order blocks A_m = 2pi Y_lm(theta_k) (k >= m rings as rows, l >= m
// degrees as columns; transform.py:416-429) depend only on the grid, and so
// does the row order that partial pivoting picks for them.  It is found once,
// on the plan's first forward call, by LU with partial pivoting (cuSOLVER
// getrf, a library factorisation used for this one-time setup only); every
// call then factors with that fixed order in the hand-written static-pivot
// kernels (factor_np.cu for n <= 256, factor_bf.cu above), which need no
// pivot search.  Gauss-Jordan with partial pivoting picks the same rows as LU
// (its extra eliminations above the diagonal do not touch the rows that are
// searched), so this is the pivot order of the reference-equivalent
// elimination (LU vs gelsy: max|df| 2.2e-14 at L=512).
#include <cusolverDn.h>

#include <vector>

#include <string>

#include "../../include/osph.h"
#include "plan.cuh"

// A_m in natural ring order, column-major: W[(l - m) * n + (k - m)].
__global__ void k_gen_block_natural(int L, int m, const double* __restrict__ costh, const double2* __restrict__ rec,
                                    const int* __restrict__ ls_tab, const double2* __restrict__ pstart,
                                    double* __restrict__ W) {
  const int n = L - m;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int k = m + i;
  const int64_t ts = (int64_t)m * L + k;
  const int ls = __ldg(ls_tab + ts);
  const double2 pp = __ldg(pstart + ts);
  double p0 = pp.x, p1 = pp.y;
  const double x = __ldg(costh + k);
  const double2* recm = rec + packed_pos(L, m, 0);
  for (int l = m; l < L; ++l) {
    double v = 0.0;
    if (l >= ls) {
      v = OSPH_TWO_PI * p1;
      const double2 ar = __ldg(recm + (l - m));
      const double nxt = fma(x, p1, -ar.x * p0) * ar.y;
      p0 = p1;
      p1 = nxt;
    }
    W[(int64_t)(l - m) * n + i] = v;
  }
}

#define CUSOLVER_TRY(expr)                                  \
  do {                                                      \
    if ((expr) != CUSOLVER_STATUS_SUCCESS) {                \
      osph_set_error(std::string("cuSOLVER: ") + #expr);    \
      rc = OSPH_ERR_CUDA;                                   \
      goto done;                                            \
    }                                                       \
  } while (0)
#define CUDA_TRY_P(expr)                                                          \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      osph_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));         \
      rc = OSPH_ERR_CUDA;                                                         \
      goto done;                                                                  \
    }                                                                             \
  } while (0)

// Fills p->d_piv (perm[packed_pos(L, m, i)] = ring offset at pivot position i)
// and sets p->piv_ready.  Host-blocking; runs on the plan stream.
int discover_pivots(osph_plan* p) {
  const int L = p->L;
  const int64_t npk = (int64_t)L * (L + 1) / 2;
  int rc = OSPH_OK;
  cusolverDnHandle_t h = nullptr;
  double* W = nullptr;
  double* work = nullptr;
  int* ipiv = nullptr;
  int* info = nullptr;
  int lwork = 0;
  std::vector<int> h_ipiv, h_perm;
  CUSOLVER_TRY(cusolverDnCreate(&h));
  CUSOLVER_TRY(cusolverDnSetStream(h, p->stream));
  CUDA_TRY_P(cudaMalloc(&W, sizeof(double) * (size_t)L * L));
  CUDA_TRY_P(cudaMalloc(&ipiv, sizeof(int) * npk));
  CUDA_TRY_P(cudaMalloc(&info, sizeof(int) * L));
  CUSOLVER_TRY(cusolverDnDgetrf_bufferSize(h, L, L, W, L, &lwork));
  CUDA_TRY_P(cudaMalloc(&work, sizeof(double) * (size_t)std::max(lwork, 1)));
  for (int m = 0; m < L; ++m) {
    const int n = L - m;
    k_gen_block_natural<<<(n + 127) / 128, 128, 0, p->stream>>>(L, m, p->d_cos, p->d_rec, p->d_ls, p->d_pstart, W);
    CUDA_TRY_P(cudaGetLastError());
    // a singular block keeps whatever order getrf reached; the factor kernels flag it
    CUSOLVER_TRY(cusolverDnDgetrf(h, n, n, W, n, work, ipiv + packed_pos(L, m, 0), info + m));
  }
  h_ipiv.resize(npk);
  CUDA_TRY_P(cudaMemcpyAsync(h_ipiv.data(), ipiv, sizeof(int) * npk, cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY_P(cudaStreamSynchronize(p->stream));
  h_perm.resize(npk);
  for (int m = 0; m < L; ++m) {  // sequential LAPACK interchanges -> pivot order
    const int n = L - m;
    int* perm = h_perm.data() + packed_pos(L, m, 0);
    const int* ip = h_ipiv.data() + packed_pos(L, m, 0);
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int i = 0; i < n; ++i) {
      const int j = ip[i] - 1;
      if (j > i && j < n) std::swap(perm[i], perm[j]);
    }
  }
  CUDA_TRY_P(cudaMemcpyAsync(p->d_piv, h_perm.data(), sizeof(int) * npk, cudaMemcpyHostToDevice, p->stream));
  CUDA_TRY_P(cudaStreamSynchronize(p->stream));
  p->piv_ready = true;
done:
  if (h) cusolverDnDestroy(h);
  cudaFree(W);
  cudaFree(work);
  cudaFree(ipiv);
  cudaFree(info);
  return rc;
}
