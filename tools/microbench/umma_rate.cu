// tcgen05.mma (kind::f16, bf16 -> f32, M=128, K=16, cta_group::1) issue rate
// for the operand layouts K7 can use: MN-major and K-major, no swizzle.
// One CTA per SM, one thread issues `iters` x 6 MMAs (commit every 6, like
// a K7 chunk) over fixed smem operands; reports TFLOP/s over the grid.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

template <int N, int MAJOR>  // MAJOR 1: MN-major, 0: K-major
__global__ void rate(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  unsigned char* a = sm;                 // 3 planes x 128 x 16 bf16
  unsigned char* b = sm + 3 * 4096;      // 3 planes x 16 x N bf16
  for (int i = threadIdx.x; i < (3 * 4096 + 3 * 32 * N) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(sa(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)MAJOR << 15) | ((uint32_t)MAJOR << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    // MN-major: LBO = K-group stride, SBO = 128 (adjacent MN groups)
    // K-major : core matrix 8 rows x 16 B, K groups adjacent (LBO = 128), SBO = MN-group stride (256 for K=16)
    const uint32_t a_lbo = MAJOR ? 2048 : 128, a_sbo = MAJOR ? 128 : 256;
    const uint32_t b_lbo = MAJOR ? (N / 8) * 128 : 128, b_sbo = MAJOR ? 128 : 256;
    unsigned long long t0 = clock64();
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const uint64_t ad = desc(sa(a) + (q % 3) * 4096, a_lbo, a_sbo);
        const uint64_t bd = desc(sa(b) + (q / 2) * 32 * N, b_lbo, b_sbo);
        const uint32_t acc = (it | q) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      if ((it & 7) == 7) {  // bounded in-flight work, like the K7 plane ring
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sa(&bar)) : "memory");
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(done) : "r"(sa(&bar)), "r"(phase) : "memory");
        phase ^= 1;
      }
    }
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(512));
}

template <int N, int MAJOR>
int run(const char* name) {
  const int iters = 4096, blocks = 148;
  unsigned long long* d;
  CK(cudaMalloc(&d, blocks * 8));
  const int smem = 3 * 4096 + 3 * 32 * N;
  CK(cudaFuncSetAttribute(rate<N, MAJOR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  rate<N, MAJOR><<<blocks, 128, smem>>>(64, d);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate<N, MAJOR><<<blocks, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * N * 16 * 6.0 * iters * blocks;
  printf("%-28s N=%3d: %8.1f TFLOP/s  %6.1f cycles per MMA (block 0)\n", name, N, flops / ms / 1e9,
         (double)h[0] / (6.0 * iters));
  cudaFree(d);
  return 0;
}

int main() {
  run<64, 1>("MN-major no-swizzle");
  run<128, 1>("MN-major no-swizzle");
  run<256, 1>("MN-major no-swizzle");
  run<64, 0>("K-major no-swizzle");
  run<128, 0>("K-major no-swizzle");
  return 0;
}
