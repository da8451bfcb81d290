// common.cuh -- shared definitions for libosph (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#define OSPH_PI 3.141592653589793238462643383279502884
#define OSPH_TWO_PI 6.283185307179586476925286766559005768

// Rescaling window of the Legendre recurrence: |mantissa| kept in
// [2^-500, 2^500], shifts of 2^1000 (pkg/src/optisph/legendre.py:31-36).
#define OSPH_BIG 0x1p500
#define OSPH_TINY 0x1p-500
#define OSPH_UP 0x1p1000
#define OSPH_DOWN 0x1p-1000

// Ring DFTs with n <= OSPH_DIRECT_MAX use a direct O(n^2) DFT; longer rings
// use Bluestein with a power-of-two FFT of size >= 2n-1 held in shared memory.
#define OSPH_DIRECT_MAX 63
#define OSPH_FFT_MAX 8192  // largest one-CTA FFT (complex double: 128 KB); 16384 runs on 2-CTA clusters
#define OSPH_SW_SMEM 2048     // per-stage FFT twiddles kept in shared memory (spans < 1024)
#define OSPH_SW_GLOBAL 16384  // global per-stage twiddle table: spans up to 4096 (N <= 16384)
// Bluestein FFTs of up to OSPH_REG_FFT_MAX points run register-resident (fft_reg.cuh);
// OSPH_RTW_SIZE: entries of their inter-pass twiddle tables (tables.cu k_reg_twiddles)
#define OSPH_REG_FFT_MAX 2048  // 2048 = two 1024-point convolutions (even / odd bins)
#define OSPH_RTW_SIZE 1872

// Position of (order m, ring/degree offset i) in order-major packed storage:
// sum_{m'<m} (L - m') + i   (same packing as transform.py:268-291 offsets).
__host__ __device__ __forceinline__ int64_t packed_pos(int L, int m, int i) {
  return (int64_t)m * L - ((int64_t)m * (m - 1)) / 2 + i;
}

// Row stride of the per-order sweep vectors w_m and u_m ([L][uw_ld(L)] doubles):
// even, so every row starts 16-byte aligned for the sweep's bulk copies.
__host__ __device__ __forceinline__ int64_t uw_ld(int L) { return (int64_t)((L + 1) & ~1); }

// Forward right-hand side / ring spectra R, TEAM-MAJOR: the maps are grouped in
// teams of G = 2^lgG (the sweep's maps per team) and a team's slab
// [pos][+-][map] is contiguous, so a team reads the right-hand side of order m
// (positions pos(m, 0..n-1)) as one block and teams working on the same order
// touch different L2 lines (no atomic hot-spotting across teams).
__host__ __device__ __forceinline__ int64_t r_index(int64_t pos, int slot, int b, int lgG, int64_t npos) {
  return ((((int64_t)(b >> lgG) * npos + pos) * 2 + slot) << lgG) + (b & ((1 << lgG) - 1));
}

// Chunk-major 8-row tiling of the sweep operands (X_m and the below-block
// Pb_m): columns are grouped in chunks of OSPH_TILE_KC, rows in tiles of 8;
// element (r, k) of a matrix with nrt row tiles lives at
//   ((k / KC) * nrt + r / 8) * KC * 8 + (k % KC) * 8 + r % 8,
// so one chunk of a contiguous row-tile range is one contiguous block (a
// single bulk copy).  Padding rows / columns are zero.
#define OSPH_TILE_KC 32
// Blocked sweep (sweep_block.cu): orders are peeled in blocks of OSPH_SB_BLOCK; order s keeps
// the coupling rows U_s[r, :] = Pb_s[s-1-r, :] X_s of the rings just below it, r < sb_rows(s)
// (every ring below s for the final block s < OSPH_SB_BLOCK), tiled like X.
#define OSPH_SB_BLOCK 32
__host__ __device__ __forceinline__ int sb_rows(int s) { return s < OSPH_SB_BLOCK ? OSPH_SB_BLOCK : OSPH_SB_BLOCK / 2; }
__host__ __device__ __forceinline__ int64_t tile_index(int r, int k, int nrt) {
  return ((((int64_t)(k >> 5)) * nrt + (r >> 3)) << 8) + ((k & 31) << 3) + (r & 7);
}
__host__ __device__ __forceinline__ int64_t tile_size(int rows, int cols) {
  return (int64_t)((cols + OSPH_TILE_KC - 1) / OSPH_TILE_KC) * ((rows + 7) / 8) * OSPH_TILE_KC * 8;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }

// m8n8k4 fp64 tensor-core MMA (SASS DMMA.8x8x4): D = A(8x4,row) * B(4x8,col) + C.
// Fragment layout (lane = 4*g + t): A[g][t], B[t][g], C/D[g][2t], C/D[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Programmatic dependent launch for the per-order kernel chains (sweep_gemm.cu,
// sweep_large.cu): each kernel lets the next one be scheduled as soon as all
// of its own CTAs have started, and waits for the previous grid (completion
// and memory) before touching data -- the launch latency of the next order
// hides under the tail of this one.
__device__ __forceinline__ void pdl_start() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

#ifdef __CUDACC__
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
#endif
