// RED.ADD.F64 completion latency seen by fence.acq_rel.gpu (B200): N reductions per thread, optional delay.
#include <cstdio>
__global__ void k(double* g, long long* cyc, int nred, int delay, int spread) {
  const int tid = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < nred; ++i) atomicAdd(g + ((size_t)(blockIdx.x * 128 + tid) * 16 + i) * spread, 1.0);
  long long t1 = clock64();
  while (clock64() - t1 < delay) {}
  long long t2 = clock64();
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  long long t3 = clock64();
  if (tid == 0) { cyc[blockIdx.x * 3] = t1 - t0; cyc[blockIdx.x * 3 + 1] = t3 - t2; }
}
int main() {
  double* g; long long* cyc; cudaMalloc(&g, 1ull << 30); cudaMalloc(&cyc, 1 << 16); cudaMemset(g, 0, 1ull << 30);
  for (int blocks : {1, 128}) for (int nred : {1, 4, 16}) for (int delay : {0, 1000, 3000}) {
    for (int it = 0; it < 3; ++it) { k<<<blocks, 128>>>(g, cyc, nred, delay, 1); cudaDeviceSynchronize(); }
    long long c[3]; cudaMemcpy(c, cyc, 24, cudaMemcpyDeviceToHost);
    printf("blocks %3d nred %2d delay %4d: issue %5lld  fence %5lld cycles\n", blocks, nred, delay, c[0], c[1]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
