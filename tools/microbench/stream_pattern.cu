// Read-bandwidth probe for K7's A stream: a column-major m x n fp32 matrix
// read in (128-row x 16-column) chunks by cp.async (16 B per lane, 8 lanes
// down a column), `depth` chunks in flight per CTA, one CTA per SM.
//   order 0: tiles round-robin over CTAs (tile = b + i * grid)   [K7 today]
//   order 1: contiguous tile ranges per CTA
//   rows   : tile height (128 | 256 | 512): more contiguous bytes per column
// plus a plain float4 grid-stride read of the same bytes as the reference.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int DEPTH, int ROWS>
__global__ void __launch_bounds__(256, 1) pattern(const float* __restrict__ a, long long m, int n, int order, float* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int kChunkBytes = ROWS * 16 * 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long ntiles = m / ROWS;
  const int nkc = n / 16;
  const long long per = (ntiles + gridDim.x - 1) / gridDim.x;
  const long long t_begin = order ? blockIdx.x * per : blockIdx.x;
  const long long t_end = order ? (t_begin + per < ntiles ? t_begin + per : ntiles) : ntiles;
  const long long t_step = order ? 1 : gridDim.x;
  long long my = 0;
  for (long long t = t_begin; t < t_end; t += t_step) ++my;
  const long long nch = my * nkc;
  // chunk: ROWS x 16 columns; 256 threads x 16 B = 4 KB per instruction round
  constexpr int kRounds = kChunkBytes / 4096;
  long long tile = t_begin;
  int kc = 0, slot = 0;
  long long g_issue = 0;
  float acc = 0.f;
  auto issue = [&]() {
    if (g_issue < nch) {
      unsigned char* dst = sm + slot * kChunkBytes;
#pragma unroll
      for (int r = 0; r < kRounds; ++r) {
        // 8 lanes x 16 B = 128 B down a column; a warp covers 4 columns x 32 rows
        const int idx = r * 256 + threadIdx.x;           // 16-byte piece id within the chunk
        const int col = idx / (ROWS / 4);                 // ROWS/4 pieces per column
        const int rp = idx - col * (ROWS / 4);
        cp16(dst + idx * 16, a + (long long)(kc * 16 + col) * m + tile * ROWS + rp * 4);
      }
      if (++kc == nkc) { kc = 0; tile += t_step; }
      if (++slot == DEPTH) slot = 0;
      ++g_issue;
    }
    commit();
  };
  for (int i = 0; i < DEPTH; ++i) issue();
  int rs = 0;
  for (long long g = 0; g < nch; ++g) {
    waitg<DEPTH - 1>();
    const float4 v = *reinterpret_cast<const float4*>(sm + rs * kChunkBytes + threadIdx.x * 16);
    acc += v.x + v.y + v.z + v.w;
    if (++rs == DEPTH) rs = 0;
    __syncwarp();
    issue();
  }
  waitg<0>();
  if (acc == 12345.f) sink[threadIdx.x] = acc;
  (void)warp; (void)lane;
}

__global__ void plain(const float4* __restrict__ a, long long n4, float* sink) {
  float acc = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = a[i];
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) sink[threadIdx.x] = acc;
}

template <int DEPTH, int ROWS>
int run(const float* a, long long m, int n, int order, float* sink) {
  const int smem = DEPTH * ROWS * 16 * 4;
  if (smem > 227 * 1024) return 0;
  CK(cudaFuncSetAttribute(pattern<DEPTH, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  pattern<DEPTH, ROWS><<<148, 256, smem>>>(a, m, n, order, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  pattern<DEPTH, ROWS><<<148, 256, smem>>>(a, m, n, order, sink);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("cp.async depth=%2d rows=%3d order=%d (smem %3d KB): %7.1f GB/s\n", DEPTH, ROWS, order, smem / 1024,
         (double)m * n * 4 / ms / 1e6);
  return 0;
}

int main() {
  const long long m = 1LL << 24;
  const int n = 128;
  float* a; float* sink;
  CK(cudaMalloc(&a, m * n * 4));
  CK(cudaMalloc(&sink, 4096));
  CK(cudaMemset(a, 0, m * n * 4));
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    plain<<<148 * 8, 256>>>(reinterpret_cast<const float4*>(a), m * n / 4, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("plain float4 grid-stride: %7.1f GB/s\n", (double)m * n * 4 / ms / 1e6);
  }
  for (int order = 0; order < 2; ++order) {
    run<4, 128>(a, m, n, order, sink);
    run<8, 128>(a, m, n, order, sink);
    run<16, 128>(a, m, n, order, sink);
    run<24, 128>(a, m, n, order, sink);
    run<4, 256>(a, m, n, order, sink);
    run<8, 256>(a, m, n, order, sink);
    run<12, 256>(a, m, n, order, sink);
    run<4, 512>(a, m, n, order, sink);
    run<6, 512>(a, m, n, order, sink);
  }
  return 0;
}
