// Rolled, rotating register-resident Gauss-Jordan panel step (as factor_np.cu): cycles per pivot.
#include <cstdio>
#define FNP_NB 32
template <int NT>
__global__ void __launch_bounds__(256, 1) k(double* out, long long* cyc, int reps, int n) {
  __shared__ __align__(16) double rowbuf[2 * FNP_NB];
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  double d[FNP_NB];
#pragma unroll
  for (int c = 0; c < FNP_NB; ++c) d[c] = (tid == c ? 40.0 : 0.0) + 1.0 / (1 + tid + c);
  const bool hasrow = tid < n;
  const int j0 = 0, nb = FNP_NB;
  auto publish = [&](double* pn) {
#pragma unroll
    for (int c = 0; c < FNP_NB - 2; c += 2) *reinterpret_cast<double2*>(pn + c) = make_double2(d[c + 1], d[c + 2]);
    if (d[0] == 0.0 || !isfinite(d[0])) s_bad = 1;
    *reinterpret_cast<double2*>(pn + FNP_NB - 2) = make_double2(d[FNP_NB - 1], 1.0 / d[0]);
  };
  double sc = 1.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (hasrow && tid == j0) publish(rowbuf);
    for (int p = 0; p < nb; ++p) {
      __syncthreads();
      const double* pr = rowbuf + (p & 1) * FNP_NB;
      double v[FNP_NB];
#pragma unroll
      for (int c = 0; c < FNP_NB; c += 2) {
        const double2 t2 = *reinterpret_cast<const double2*>(pr + c);
        v[c] = t2.x;
        v[c + 1] = t2.y;
      }
      const double inv = v[FNP_NB - 1];
      if (hasrow) {
        // lazy pivot scaling: the pivot row only rotates (gg = 0, new column 1)
        // and remembers its scale 1/piv, applied once after the panel
        const bool ispiv = tid == j0 + p;
        const bool nextpub = p + 1 < nb && tid == j0 + p + 1;
        const double gg = ispiv ? 0.0 : d[0] * inv;
        sc = ispiv ? inv : sc;
        const double nd0 = fma(-gg, v[0], d[1]);  // the next pivot first: its reciprocal starts early
        double rn = 0.0;
        if (nextpub) rn = 1.0 / nd0;
        d[0] = nd0;
#pragma unroll
        for (int c = 1; c < FNP_NB - 1; ++c) d[c] = fma(-gg, v[c], d[c + 1]);
        d[FNP_NB - 1] = ispiv ? 1.0 : -gg;
        if (nextpub) {
          double* pn = rowbuf + ((p + 1) & 1) * FNP_NB;
#pragma unroll
          for (int c = 0; c < FNP_NB - 2; c += 2) *reinterpret_cast<double2*>(pn + c) = make_double2(d[c + 1], d[c + 2]);
          if (nd0 == 0.0 || !isfinite(nd0)) s_bad = 1;
          *reinterpret_cast<double2*>(pn + FNP_NB - 2) = make_double2(d[FNP_NB - 1], rn);
        }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < FNP_NB; ++c) s += d[c];
  out[blockIdx.x * blockDim.x + tid] = s * sc + s_bad;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1024);
  const int reps = 50;
  for (int n : {32, 64, 128, 256}) {
    for (int it = 0; it < 2; ++it) { k<256><<<1, 256>>>(out, cyc, reps, n); cudaDeviceSynchronize(); }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("n=%d (256 threads): %.1f cycles per pivot step\n", n, (double)c / (reps * FNP_NB));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
