// Read+write bandwidth probe for K7's access pattern without the math: every
// CTA (one per SM) streams 128-row (or ROWS-row) tiles of a column-major
// m x n fp32 A through a cp.async staging ring and writes the same tile to U
// (column-major, same shape), the way K7 reads A and writes U.
//   W0: thread = row, one STG.32 per column (K7's epilogue today)
//   W1: thread = 4 consecutive rows, STG.128 per column (4x fewer stores)
// plus a plain float4 grid-stride copy as the reference.
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

// chunk = ROWS x 16 columns; DEPTH chunks in flight; 256 threads
template <int DEPTH, int ROWS, int WMODE>
__global__ void __launch_bounds__(256, 1) copy_k(const float* __restrict__ a, float* __restrict__ u, long long m, int n) {
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int kChunkBytes = ROWS * 16 * 4;
  constexpr int kRounds = kChunkBytes / 4096;
  const long long ntiles = m / ROWS;
  const int nkc = n / 16;
  long long my = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) ++my;
  const long long nch = my * nkc;
  long long tile_i = blockIdx.x;
  int kc_i = 0, slot = 0;
  long long g_issue = 0;
  auto issue = [&]() {
    if (g_issue < nch) {
      unsigned char* dst = sm + slot * kChunkBytes;
#pragma unroll
      for (int r = 0; r < kRounds; ++r) {
        const int idx = r * 256 + threadIdx.x;
        const int col = idx / (ROWS / 4);
        const int rp = idx - col * (ROWS / 4);
        cp16(dst + idx * 16, a + (long long)(kc_i * 16 + col) * m + tile_i * ROWS + rp * 4);
      }
      if (++kc_i == nkc) { kc_i = 0; tile_i += gridDim.x; }
      if (++slot == DEPTH) slot = 0;
      ++g_issue;
    }
    commit();
  };
  for (int i = 0; i < DEPTH; ++i) issue();
  int rs = 0;
  long long tile = blockIdx.x;
  int kc = 0;
  for (long long g = 0; g < nch; ++g) {
    waitg<DEPTH - 1>();
    __syncthreads();
    const float* src = reinterpret_cast<const float*>(sm + rs * kChunkBytes);
    if (WMODE == 0) {
      // thread = row (ROWS / 256 rows per thread), STG.32 per column
      for (int rr = threadIdx.x; rr < ROWS; rr += 256) {
        float* dst = u + (long long)(kc * 16) * m + tile * ROWS + rr;
#pragma unroll
        for (int c = 0; c < 16; ++c) dst[(long long)c * m] = src[c * ROWS + rr];
      }
    } else {
      // thread = 4 rows, STG.128 per column
      for (int q = threadIdx.x; q < ROWS / 4; q += 256) {
        float* dst = u + (long long)(kc * 16) * m + tile * ROWS + 4 * q;
#pragma unroll
        for (int c = 0; c < 16; ++c)
          *reinterpret_cast<float4*>(dst + (long long)c * m) = *reinterpret_cast<const float4*>(src + c * ROWS + 4 * q);
      }
      // ROWS / 4 < 256: the remaining threads idle
    }
    __syncthreads();
    if (++rs == DEPTH) rs = 0;
    if (++kc == nkc) { kc = 0; tile += gridDim.x; }
    issue();
  }
  waitg<0>();
}

__global__ void plain_copy(const float4* __restrict__ a, float4* __restrict__ u, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    u[i] = a[i];
}

template <int DEPTH, int ROWS, int WMODE>
int run(const float* a, float* u, long long m, int n) {
  const int smem = DEPTH * ROWS * 16 * 4;
  if (smem > 227 * 1024) return 0;
  CK(cudaFuncSetAttribute(copy_k<DEPTH, ROWS, WMODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  copy_k<DEPTH, ROWS, WMODE><<<148, 256, smem>>>(a, u, m, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  copy_k<DEPTH, ROWS, WMODE><<<148, 256, smem>>>(a, u, m, n);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("tile copy depth=%2d rows=%3d W%d: %7.1f GB/s (read+write)\n", DEPTH, ROWS, WMODE, 2.0 * m * n * 4 / ms / 1e6);
  return 0;
}

int main() {
  const long long m = 1LL << 24;
  const int n = 128;
  float *a, *u;
  CK(cudaMalloc(&a, m * n * 4));
  CK(cudaMalloc(&u, m * n * 4));
  CK(cudaMemset(a, 0, m * n * 4));
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    plain_copy<<<148 * 8, 256>>>(reinterpret_cast<const float4*>(a), reinterpret_cast<float4*>(u), m * n / 4);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("plain float4 copy: %7.1f GB/s (read+write)\n", 2.0 * m * n * 4 / ms / 1e6);
  }
  run<8, 128, 0>(a, u, m, n);
  run<16, 128, 0>(a, u, m, n);
  run<8, 256, 0>(a, u, m, n);
  run<8, 512, 0>(a, u, m, n);
  run<16, 128, 1>(a, u, m, n);
  run<8, 256, 1>(a, u, m, n);
  run<8, 512, 1>(a, u, m, n);
  run<6, 1024, 1>(a, u, m, n);
  return 0;
}
