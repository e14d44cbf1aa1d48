// Write-bandwidth probe for K7's U epilogue: 148 CTAs x 4 warps store a
// column-major m x n fp32 matrix in 128-row tiles (round-robin over CTAs).
//   S1: each thread owns one row; STG.32 per column (128 B per warp instr)
//   S2: tile staged in smem, then STG.128 down the columns (512 B per instr)
//   S3: tile staged in smem, one thread issues 512-B bulk copies smem->global
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int MODE>
__global__ void __launch_bounds__(128, 1) store_k(float* __restrict__ u, long long m, int n) {
  extern __shared__ __align__(128) float st[];  // [2][n][128 + 4]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long ntiles = m / 128;
  int buf = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long row0 = t * 128;
    if (MODE == 0) {
      const long long row = row0 + threadIdx.x;
      for (int c = 0; c < n; ++c) u[(long long)c * m + row] = (float)(c + row);
    } else {
      float* s = st + buf * n * 132;
      if (MODE == 2) {  // make sure the bulk reads of this buffer (2 tiles ago) are done
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
        __syncthreads();
      }
      for (int c = 0; c < n; ++c) s[c * 132 + threadIdx.x] = (float)(c + row0 + threadIdx.x);
      if (MODE == 2) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncthreads();
      if (MODE == 1) {
        // warp w stores columns w, w+4, ...: 32 lanes x 16 B = 512 B per column
        for (int c = warp; c < n; c += 4) {
          const float4 v = *reinterpret_cast<const float4*>(s + c * 132 + lane * 4);
          *reinterpret_cast<float4*>(u + (long long)c * m + row0 + lane * 4) = v;
        }
        __syncthreads();
      } else {
        if (threadIdx.x == 0) {
          for (int c = 0; c < n; ++c)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;\n" ::"l"(u + (long long)c * m + row0),
                         "r"((unsigned)__cvta_generic_to_shared(s + c * 132))
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
      }
      buf ^= 1;
    }
  }
  if (MODE == 2 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

template <int MODE>
int run(float* u, long long m, int n, const char* name) {
  const int smem = MODE ? 2 * n * 132 * 4 : 0;
  CK(cudaFuncSetAttribute(store_k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  store_k<MODE><<<148, 128, smem>>>(u, m, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  store_k<MODE><<<148, 128, smem>>>(u, m, n);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-40s n=%3d: %7.1f GB/s\n", name, n, (double)m * n * 4 / ms / 1e6);
  return 0;
}

int main() {
  const long long m = 1LL << 24;
  float* u;
  CK(cudaMalloc(&u, m * 128 * 4));
  for (int n : {64, 128}) {
    run<0>(u, m, n, "S1 STG.32 per column (row per thread)");
    run<1>(u, m, n, "S2 smem transpose + STG.128");
    run<2>(u, m, n, "S3 smem + 512-B bulk stores");
  }
  return 0;
}
