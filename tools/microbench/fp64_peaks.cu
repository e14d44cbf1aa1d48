// Microbenchmarks that size the design: DFMA vs DMMA (mma.sync f64) peak,
// FFMA peak, cooperative grid.sync latency, fp64 div/sqrt latency.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.0f) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void gridsync_kernel(int iters, unsigned long long* t) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) t[0] = clock64() - t0;
}

__global__ void divsqrt_latency(double* out, int iters, double x) {
  double v = x;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = 1.0 / sqrt(v + 1.0) + 1.0;
  unsigned long long t1 = clock64();
  out[0] = v;
  out[1] = (double)(t1 - t0) / iters;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("device %s sms=%d clock=%d kHz\n", p.name, sms, p.clockRate);
  double* d; float* f; unsigned long long* t;
  CK(cudaMalloc(&d, 64)); CK(cudaMalloc(&f, 64)); CK(cudaMalloc(&t, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int iters = 20000;
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    dfma_kernel<8><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
  }
  for (int threads : {256, 512}) {
    int blocks = sms * (2048 / threads);
    ffma_kernel<8><<<blocks, threads>>>(f, 100, 1.0000001f, 1e-9f);
    cudaEventRecord(e0);
    ffma_kernel<8><<<blocks, threads>>>(f, iters, 1.0000001f, 1e-9f);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf("FFMA threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) {
    int blocks = sms * (2048 / threads);
    dmma_kernel<4><<<blocks, threads>>>(d, 100);
    cudaEventRecord(e0);
    dmma_kernel<4><<<blocks, threads>>>(d, iters / 4);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 4 * (iters / 4) * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4 threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
  }
  for (int nb : {1, 8, 37, 74, 148}) {
    int it = 2000;
    void* args[] = {&it, &t};
    CK(cudaLaunchCooperativeKernel((void*)gridsync_kernel, nb, 256, args, 0, 0));
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)gridsync_kernel, nb, 256, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("grid.sync blocks=%d: %.3f us/sync\n", nb, ms * 1e3 / it);
  }
  divsqrt_latency<<<1, 1>>>(d, 1000, 2.0);
  double h[2];
  CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
  printf("fp64 1/sqrt(x+1)+1 dependent chain: %.1f cycles/iter\n", h[1]);
  return 0;
}
