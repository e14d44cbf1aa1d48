// Latency of one fp64 Jacobi rotation (the formula of csrc/jacobi.cu) for one
// warp, dependent chain, vs the pieces (sqrt, div) on their own.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "common.cuh"

__device__ __noinline__ void rescale(double& x, double& y, double big) {
  int e;
  frexp(big, &e);
  x = ldexp(x, -e);
  y = ldexp(y, -e);
}

__global__ void rot_chain(double* out, int iters, double tol) {
  double app = 2.0 + threadIdx.x * 1e-3, aqq = 1.0, apq = 0.25;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double pr = app * aqq;
    const double thresh = (pr > 0x1p-1000 && pr < 0x1p1000) ? tol * sqrt(pr) : tol * sqrt(app) * sqrt(aqq);
    const bool act = !(fabs(apq) <= thresh);
    double x = aqq - app, y = 2.0 * apq;
    const bool xzero = x == 0.0, xpos = x > 0.0;
    const double big = fmax(fabs(x), fabs(y));
    if (!(big < 0x1p500 && big > 0x1p-500)) rescale(x, y, big);
    const double ax = fabs(x);
    const double q = fma(x, x, y * y);
    const double ys = xpos ? y : -y;
    double t, c;
    if (big < 0x1p400 && big > 0x1p-400 && fabs(y) > big * 0x1p-200) {
      const double r = mpsvd::dev::fast_sqrt_normal(q), iq = mpsvd::dev::fast_div_normal(1.0, q);
      const double den = ax + r;
      t = xzero ? 1.0 : mpsvd::dev::fast_div_normal(ys, den);
      c = mpsvd::dev::fast_sqrt_normal(fma(0.5, ax * (r * iq), 0.5));
    } else {
      const double r = sqrt(q), iq = 1.0 / q;
      const double den = ax + r;
      t = xzero ? 1.0 : ys / den;
      c = sqrt(fma(0.5, ax * (r * iq), 0.5));
    }
    const double s = c * t;
    // feed back so iterations are dependent
    app = 2.0 + s * 1e-9 + (act ? 0.0 : 1e-300);
    apq = 0.25 + c * 1e-9;
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / iters; out[1] = app + apq; }
}

__global__ void sqrt_chain(double* out, int iters) {
  double v = 2.0 + threadIdx.x;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = sqrt(v) + 1.0;
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / iters; out[1] = v; }
}

__global__ void div_chain(double* out, int iters) {
  double v = 2.0 + threadIdx.x;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = 3.0 / v + 1.0;
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / iters; out[1] = v; }
}

__global__ void dfma_chain(double* out, int iters) {
  double v = 2.0 + threadIdx.x;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = fma(v, 0.999, 1e-3);
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / iters; out[1] = v; }
}

// one 512-thread block: dependent __syncthreads hand-offs (a value written
// by one warp is read by another after every barrier)
__global__ void sync_chain(double* out, int iters) {
  __shared__ volatile int flag[2];
  if (threadIdx.x == 0) flag[0] = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == (unsigned)((i & 15) * 32)) flag[i & 1] = flag[(i + 1) & 1] + 1;
    __syncthreads();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / iters; out[1] = flag[0]; }
}

// cooperative grid barrier, one 512-thread CTA per SM (the multi-CTA solver's shape)
__global__ void grid_chain(double* out, int iters) {
  namespace cg = cooperative_groups;
  cg::grid_group g = cg::this_grid();
  g.sync();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
}

// the multi-CTA solver's own barrier (csrc/jacobi.cu garrive / gwait): a
// monotonic arrival counter, one atomic per CTA, thread 0 polls with acquire
__global__ void grid_chain_counter(double* out, int iters, unsigned* bar) {
  unsigned seq = 0;
  auto sync = [&]() {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1u);
    }
    ++seq;
    if (threadIdx.x == 0) {
      const unsigned target = seq * gridDim.x;
      unsigned seen;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(seen) : "l"(bar) : "memory");
      } while ((int)(seen - target) < 0);
    }
    __syncthreads();
  };
  sync();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) sync();
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
}

int main() {
  double* d;
  cudaMalloc(&d, 16);
  double h[2];
  const int it = 2000;
  rot_chain<<<1, 32>>>(d, it, 64 * 0x1p-53);
  rot_chain<<<1, 32>>>(d, it, 64 * 0x1p-53);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("rotation chain: %.1f cycles/rotation\n", h[0]);
  sqrt_chain<<<1, 32>>>(d, it);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("sqrt+add chain: %.1f cycles\n", h[0]);
  div_chain<<<1, 32>>>(d, it);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("div+add chain: %.1f cycles\n", h[0]);
  dfma_chain<<<1, 32>>>(d, it);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("dfma chain: %.1f cycles\n", h[0]);
  double rot = 0;
  rot_chain<<<1, 32>>>(d, it, 64 * 0x1p-53);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  rot = h[0];
  sync_chain<<<1, 512>>>(d, it);
  sync_chain<<<1, 512>>>(d, it);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double syn = h[0];
  printf("__syncthreads hand-off (512 threads): %.1f cycles\n", syn);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int git = 500;
  void* args[] = {&d, &git};
  cudaLaunchCooperativeKernel((void*)grid_chain, sms, 512, args, 0, nullptr);
  cudaLaunchCooperativeKernel((void*)grid_chain, sms, 512, args, 0, nullptr);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double gs = h[0];
  printf("cg grid.sync (%d CTAs x 512): %.1f cycles\n", sms, gs);
  unsigned* bar;
  cudaMalloc(&bar, 4);
  cudaMemset(bar, 0, 4);
  void* cargs[] = {&d, &git, &bar};
  cudaLaunchCooperativeKernel((void*)grid_chain_counter, sms, 512, cargs, 0, nullptr);
  cudaMemset(bar, 0, 4);
  cudaLaunchCooperativeKernel((void*)grid_chain_counter, sms, 512, cargs, 0, nullptr);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double gc = h[0];
  printf("counter grid barrier (%d CTAs x 512): %.1f cycles\n", sms, gc);
  printf("JSON {\"rotation_chain_cycles\": %.1f, \"syncthreads_cycles\": %.1f, \"grid_sync_cycles\": %.1f, "
         "\"cg_grid_sync_cycles\": %.1f, \"sms\": %d, \"source\": \"tools/microbench/rot_latency.cu\"}\n",
         rot, syn, gc, gs, sms);
  return 0;
}
