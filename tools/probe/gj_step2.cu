// Which part of a register-resident Gauss-Jordan pivot step costs what (B200).
#include <cstdio>
#include <utility>
#include <type_traits>
#define NB 32
template <int MODE>  // bit0: row loads + FMAs, bit1: reciprocal, bit2: publish stores, bit3: selects for pivot row
__global__ void k(double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double rowbuf[2 * (NB + 2)];
  const int tid = threadIdx.x;
  double d[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) d[c] = (tid == c ? 4.0 : 0.0) + 1.0 / (1 + tid + c);
  if (tid < 2 * (NB + 2)) rowbuf[tid] = 0.5;
  auto step = [&](auto pc) {
    constexpr int p = decltype(pc)::value;
    __syncthreads();
    const double* pr = rowbuf + (p & 1) * (NB + 2);
    const double inv = pr[NB];
    const bool ispiv = tid == p;
    const double gg = d[p] * inv;
    const double mlt = (MODE & 8) ? (ispiv ? inv : -gg) : -gg;
    if (MODE & 1) {
#pragma unroll
      for (int c = 0; c < NB; c += 2) {
        const double2 v = *reinterpret_cast<const double2*>(pr + c);
        if (MODE & 8) {
          d[c] = (c == p) ? mlt : fma(mlt, ispiv ? d[c] : v.x, ispiv ? 0.0 : d[c]);
          d[c + 1] = (c + 1 == p) ? mlt : fma(mlt, ispiv ? d[c + 1] : v.y, ispiv ? 0.0 : d[c + 1]);
        } else {
          d[c] = (c == p) ? mlt : fma(mlt, v.x, d[c]);
          d[c + 1] = (c + 1 == p) ? mlt : fma(mlt, v.y, d[c + 1]);
        }
      }
    }
    double inv1 = 0.5;
    if (MODE & 2) inv1 = 1.0 / (d[(p + 1) % NB] + 2.0);
    if (MODE & 4) {
      if (tid == p + 1) {
        double* pn = rowbuf + ((p + 1) & 1) * (NB + 2);
#pragma unroll
        for (int c = 0; c < NB; c += 2) *reinterpret_cast<double2*>(pn + c) = make_double2(d[c] * 1e-3, d[c + 1] * 1e-3);
        pn[NB] = inv1 * 1e-3 + 0.5;
      }
    } else {
      d[0] += inv1 * 1e-30;
    }
  };
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    [&]<int... P>(std::integer_sequence<int, P...>) { (step(std::integral_constant<int, P>{}), ...); }(
        std::make_integer_sequence<int, NB>{});
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < NB; ++c) s += d[c];
  out[blockIdx.x * blockDim.x + tid] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int M> void run(double* out, long long* cyc, int nt) {
  const int reps = 50;
  for (int it = 0; it < 2; ++it) { k<M><<<1, nt>>>(out, cyc, reps); cudaDeviceSynchronize(); }
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("threads %3d mode %2d: %.1f cycles per step\n", nt, M, (double)c / (reps * NB));
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1024);
  for (int nt : {32, 128, 256}) {
    run<0>(out, cyc, nt); run<1>(out, cyc, nt); run<2>(out, cyc, nt); run<3>(out, cyc, nt);
    run<7>(out, cyc, nt); run<15>(out, cyc, nt);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
