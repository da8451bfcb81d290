// Standalone check of fft2.cuh's bluestein_conv2 against a direct O(N^2) circular convolution.
#include <cstdio>
#include <cmath>
#include <vector>
#include <complex>
#include "../experimental/fft2.cuh"  // register-blocked Bluestein (measured slower than the radix-4 path, kept for reference)
template <int N1, int N2>
__global__ void k(const double2* x, const double2* bh, const double2* tw, double2* out) {
  __shared__ double2 sm[conv2_stride<N1, N2>()];
  constexpr int N = N1 * N2, TPM = conv2_tpm<N1, N2>();
  for (int i = threadIdx.x; i < N; i += blockDim.x) sm[i] = x[i];
  __syncthreads();
  bluestein_conv2<N1, N2>(sm, threadIdx.x, threadIdx.x < TPM, bh, tw);
  for (int i = threadIdx.x; i < N; i += blockDim.x) out[i] = sm[i];
}
template <int N1, int N2> void run(const double2* dtw) {
  constexpr int N = N1 * N2;
  std::vector<double2> x(N), bh(N), out(N);
  for (int i = 0; i < N; ++i) { x[i] = make_double2(sin(1.3 * i), cos(0.7 * i * i)); bh[i] = make_double2(cos(0.11 * i), sin(0.5 * i)); }
  double2 *dx, *db, *dout; cudaMalloc(&dx, N * 16); cudaMalloc(&db, N * 16); cudaMalloc(&dout, N * 16);
  cudaMemcpy(dx, x.data(), N * 16, cudaMemcpyHostToDevice); cudaMemcpy(db, bh.data(), N * 16, cudaMemcpyHostToDevice);
  k<N1, N2><<<1, 64>>>(dx, db, dtw, dout);
  cudaMemcpy(out.data(), dout, N * 16, cudaMemcpyDeviceToHost);
  // reference: X = DFT(x); Z = X * bh; out = IDFT(Z) (unnormalised)
  std::vector<std::complex<double>> X(N), Z(N);
  for (int kk = 0; kk < N; ++kk) { std::complex<double> s = 0; for (int n = 0; n < N; ++n) s += std::complex<double>(x[n].x, x[n].y) * std::polar(1.0, -2 * M_PI * (double)((long)kk * n % N) / N); X[kk] = s * std::complex<double>(bh[kk].x, bh[kk].y); }
  double err = 0, mx = 0;
  for (int j = 0; j < N; ++j) { std::complex<double> s = 0; for (int kk = 0; kk < N; ++kk) s += X[kk] * std::polar(1.0, 2 * M_PI * (double)((long)kk * j % N) / N); err = fmax(err, std::abs(s - std::complex<double>(out[j].x, out[j].y))); mx = fmax(mx, std::abs(s)); }
  printf("N1=%d N2=%d: max err %.3e (max |ref| %.3e)  %s\n", N1, N2, err, mx, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  std::vector<double2> tw(16384);
  for (int j = 0; j < 16384; ++j) tw[j] = make_double2(cos(2 * M_PI * j / 16384), -sin(2 * M_PI * j / 16384));
  double2* dtw; cudaMalloc(&dtw, 16384 * 16); cudaMemcpy(dtw, tw.data(), 16384 * 16, cudaMemcpyHostToDevice);
  run<4, 4>(dtw); run<8, 4>(dtw); run<16, 16>(dtw); run<32, 16>(dtw); run<32, 32>(dtw);
}
