// Cluster-barrier cost on B200: plain, with global REDs outstanding, with DSMEM stores, relaxed.
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
template <int MODE>  // 0 plain release/acquire, 1 + REDs before arrive, 2 relaxed, 3 + DSMEM stores, 4 + global stores
__global__ void __cluster_dims__(4, 1, 1) k(double* g, long long* cyc, int iters) {
  __shared__ double sh[1024];
  const int tid = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 1) atomicAdd(g + (blockIdx.x * 256 + tid) * 8, 1.0);
    if (MODE == 3) { double* r = cg::this_cluster().map_shared_rank(sh, (cg::this_cluster().block_rank() + 1) & 3); r[tid] = i; }
    if (MODE == 4) g[(blockIdx.x * 256 + tid) * 8 + 1] = i;
    if (MODE == 2) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    else asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int M> void run(double* g, long long* cyc, int nblk) {
  const int iters = 1000;
  for (int it = 0; it < 2; ++it) { k<M><<<nblk, 256>>>(g, cyc, iters); cudaDeviceSynchronize(); }
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("mode %d, %d CTAs: %.0f cycles per barrier\n", M, nblk, (double)c / iters);
}
int main() {
  double* g; long long* cyc; cudaMalloc(&g, 64 << 20); cudaMalloc(&cyc, 4096); cudaMemset(g, 0, 64 << 20);
  for (int nb : {4, 128}) { run<0>(g, cyc, nb); run<1>(g, cyc, nb); run<2>(g, cyc, nb); run<3>(g, cyc, nb); run<4>(g, cyc, nb); }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
