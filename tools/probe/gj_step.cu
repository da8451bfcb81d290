// Microbenchmark: cycles per pivot step of the register-resident panel
// elimination (factor_np.cu), one CTA of 256 threads, 32 pivots per panel.
#include <cstdio>
#include <utility>
#include <type_traits>
#define NB 32
template <int MODE>
__global__ void k(double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double rowbuf[2 * (NB + 2)];
  const int tid = threadIdx.x;
  double d[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) d[c] = (tid == c ? 4.0 : 0.0) + 1.0 / (1 + tid + c);
  const int j0 = 0, nb = NB;
  // Divergence-free step: every thread runs the same instructions (the pivot
  // row's scaling folded into the FMA by selects), every thread computes the
  // reciprocal of its next-pivot entry, only the next pivot's thread stores.
  auto step = [&](auto pc) {
    constexpr int p = decltype(pc)::value;
    if (p >= nb) return;
    __syncthreads();
    const double* pr = rowbuf + (p & 1) * (NB + 2);
    const double inv = pr[NB];
    const bool ispiv = tid == j0 + p;
    const double gg = d[p] * inv;
    const double mlt = ispiv ? inv : -gg;
    // next pivot column first (its reciprocal is on the critical path)
    if constexpr (p + 1 < NB) d[p + 1] = fma(mlt, ispiv ? d[p + 1] : pr[p + 1], ispiv ? 0.0 : d[p + 1]);
    const double inv1 = (p + 1 < NB) ? 1.0 / d[(p + 1) % NB] : 0.0;
#pragma unroll
    for (int c = 0; c < NB; c += 2) {
      const double2 v = *reinterpret_cast<const double2*>(pr + c);
      if (c != p + 1) d[c] = (c == p) ? mlt : fma(mlt, ispiv ? d[c] : v.x, ispiv ? 0.0 : d[c]);
      if (c + 1 != p + 1) d[c + 1] = (c + 1 == p) ? mlt : fma(mlt, ispiv ? d[c + 1] : v.y, ispiv ? 0.0 : d[c + 1]);
    }
    if constexpr (p + 1 < NB) {
      if (p + 1 < nb && tid == j0 + p + 1) {
        double* pn = rowbuf + ((p + 1) & 1) * (NB + 2);
#pragma unroll
        for (int c = 0; c < NB; c += 2) *reinterpret_cast<double2*>(pn + c) = make_double2(d[c], d[c + 1]);
        pn[NB] = inv1;
      }
    }
  };
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (tid == j0) {
      for (int c = 0; c < NB; c += 2) *reinterpret_cast<double2*>(rowbuf + c) = make_double2(d[c], d[c + 1]);
      rowbuf[NB] = 1.0 / d[0];
    }
    [&]<int... P>(std::integer_sequence<int, P...>) { (step(std::integral_constant<int, P>{}), ...); }(
        std::make_integer_sequence<int, NB>{});
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < NB; ++c) s += d[c];
  out[blockIdx.x * blockDim.x + tid] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1024);
  const int reps = 100;
  for (int mode = 0; mode < 2; ++mode) {
    for (int it = 0; it < 2; ++it) {
      if (mode == 0) k<0><<<1, 256>>>(out, cyc, reps); else k<1><<<1, 256>>>(out, cyc, reps);
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %.1f cycles per pivot step\n", mode, mode ? "__drcp_rn" : "1.0/x", (double)c / (reps * NB));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
