// Latency probes on B200: dependent DFMA, division, __drcp_rn, LDS chain, bar.sync, shfl.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0) {
  __shared__ double sh[64];
  const int tid = threadIdx.x;
  double x = x0 + tid * 1e-9, y = 1.0;
  sh[tid & 63] = 1.0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) y = fma(y, x, 1e-3);
  long long t1 = clock64();
  for (int i = 0; i < 256; ++i) y = 1.0 / (y + 1.5);
  long long t2 = clock64();
  for (int i = 0; i < 256; ++i) y = __drcp_rn(y + 1.5);
  long long t3 = clock64();
  int idx = tid & 63;
  for (int i = 0; i < 256; ++i) { double v = sh[idx]; idx = ((int)v + i) & 63; y += v; }
  long long t4 = clock64();
  for (int i = 0; i < 256; ++i) __syncthreads();
  long long t5 = clock64();
  for (int i = 0; i < 256; ++i) y = __shfl_sync(0xffffffffu, y, (i + 1) & 31) * 1.0000001;
  long long t6 = clock64();
  out[tid] = y + idx;
  if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 16); cudaMalloc(&cyc, 64);
  for (int nt : {32, 256}) {
    for (int it = 0; it < 2; ++it) { k<<<1, nt>>>(out, cyc, 0.999); cudaDeviceSynchronize(); }
    long long c[6]; cudaMemcpy(c, cyc, 48, cudaMemcpyDeviceToHost);
    printf("threads %d: dfma %.1f  div %.1f  drcp %.1f  lds-chain %.1f  bar.sync %.1f  shfl+dmul %.1f cycles each\n", nt,
           c[0] / 256.0, c[1] / 256.0, c[2] / 256.0, c[3] / 256.0, c[4] / 256.0, c[5] / 256.0);
  }
}
