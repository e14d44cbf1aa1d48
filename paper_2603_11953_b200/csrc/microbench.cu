// Live fp64 peak probe: the roofline denominator for the Gram (MEASURED_PEAKS.json
// carries no fp64 figure). DMMA m8n8k4 issue-bound loop, 4 independent
// accumulator chains per warp, all SMs; reports TFLOP/s (2 flops per FMA).
#include "common.cuh"
#include "kernels.h"

namespace mpsvd {
namespace dev {

__global__ void dmma_peak_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}

double measure_fp64_peak_tflops(int device) {
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return 0.0;
  double* d = nullptr;
  if (cudaMalloc(&d, 64) != cudaSuccess) return 0.0;
  const int threads = 256, blocks = p.multiProcessorCount * 8, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_peak_kernel<<<blocks, threads>>>(d, 64);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    dmma_peak_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double flops = 2.0 * 256 * 4 * (double)iters * blocks * (threads / 32);
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace dev
}  // namespace mpsvd
