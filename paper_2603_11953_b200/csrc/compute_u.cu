// K7: U = A * (V Sigma^-1) in working precision.
//
// Reference semantics: matmul(a, scale_columns(v, sigma, invert))
// (proj/src/thinsvd.cpp:110-113, proj/src/dense.cpp:83-96,214-232): W is
// formed first (true division, done by finish_columns in jacobi.cu, stored
// row-major "W^T" so every CTA stages it with straight coalesced copies),
// then every U entry accumulates A(i,l)*W(l,j) over ascending l. Here each
// entry is one fma chain over ascending l (the reference's x86 build rounds
// the product and the sum separately; both are the same order).
//
// Tiling: a CTA owns BM=128 rows x NB output columns; A and W^T are staged
// through shared memory in BK=32 slices with a register prefetch of the next
// slice; each thread keeps a TM x TN register tile. A is streamed exactly
// once per column block (once in total for n <= NB) and U written once.
#include "common.cuh"
#include "kernels.h"

namespace mpsvd {
namespace dev {

constexpr int kBM = 128;
constexpr int kBK = 32;

template <typename T, int NB, int TM, int TN>
__global__ void __launch_bounds__(256)
av_kernel(const T* __restrict__ a, long long lda, long long m, int n, const T* __restrict__ wt,
          T* __restrict__ u, long long ldu, const DevStatus* __restrict__ status) {
  static_assert((kBM / TM) * (NB / TN) == 256, "256 threads");
  if (status && status->status != kOk) return;
  extern __shared__ __align__(16) unsigned char avsm[];
  T* as = reinterpret_cast<T*>(avsm);  // [2][kBK][kBM]
  T* ws = as + 2 * kBK * kBM;          // [2][kBK][NB]
  const int tid = threadIdx.x;
  const int tx = tid % (NB / TN), ty = tid / (NB / TN);
  const long long r0 = (long long)blockIdx.x * kBM;
  const int c0 = blockIdx.y * NB;

  constexpr int kAPer = kBK * kBM / 256;  // 16
  constexpr int kWPer = kBK * NB / 256;   // NB/8
  T pa[kAPer], pw[kWPer];
  auto load = [&](int l0) {
#pragma unroll
    for (int it = 0; it < kAPer; ++it) {
      const int e = it * 256 + tid;
      const int kk = e / kBM, i = e % kBM;
      const long long row = r0 + i;
      const int l = l0 + kk;
      pa[it] = (row < m && l < n) ? a[(long long)l * lda + row] : T(0);
    }
#pragma unroll
    for (int it = 0; it < kWPer; ++it) {
      const int e = it * 256 + tid;
      const int kk = e / NB, j = e % NB;
      const int l = l0 + kk, col = c0 + j;
      pw[it] = (l < n && col < n) ? wt[(long long)l * n + col] : T(0);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int it = 0; it < kAPer; ++it) {
      const int e = it * 256 + tid;
      as[buf * kBK * kBM + e] = pa[it];
    }
#pragma unroll
    for (int it = 0; it < kWPer; ++it) {
      const int e = it * 256 + tid;
      ws[buf * kBK * NB + e] = pw[it];
    }
  };

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  const int nchunks = (n + kBK - 1) / kBK;
  load(0);
  store(0);
  __syncthreads();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int cur = ch & 1;
    const bool more = ch + 1 < nchunks;
    if (more) load((ch + 1) * kBK);
    const T* ac = as + cur * kBK * kBM;
    const T* wc = ws + cur * kBK * NB;
    const int kmax = min(kBK, n - ch * kBK);
    for (int k = 0; k < kmax; ++k) {
      T av[TM], wv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = ac[k * kBM + ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) wv[j] = wc[k * NB + tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i], wv[j], acc[i][j]);
    }
    if (more) store(cur ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    const int col = c0 + tx * TN + j;
    if (col >= n) continue;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const long long row = r0 + ty * TM + i;
      if (row < m) u[(long long)col * ldu + row] = acc[i][j];
    }
  }
}

template <typename T, int NB, int TM, int TN>
static cudaError_t launch_av_t(const T* a, long long lda, long long m, int n, const T* w, T* u,
                               long long ldu, const DevStatus* status, cudaStream_t st) {
  auto k = av_kernel<T, NB, TM, TN>;
  const size_t smem = 2 * (size_t)kBK * (kBM + NB) * sizeof(T);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)((m + kBM - 1) / kBM), (unsigned)((n + NB - 1) / NB));
  k<<<grid, 256, smem, st>>>(a, lda, m, n, w, u, ldu, status);
  return cudaGetLastError();
}

cudaError_t launch_av_f32(const float* a, long long lda, long long m, int n, const float* w,
                          float* u, long long ldu, const DevStatus* status, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  if (n <= 32) return launch_av_t<float, 32, 4, 4>(a, lda, m, n, w, u, ldu, status, st);
  if (n <= 64) return launch_av_t<float, 64, 8, 4>(a, lda, m, n, w, u, ldu, status, st);
  return launch_av_t<float, 128, 8, 8>(a, lda, m, n, w, u, ldu, status, st);
}

cudaError_t launch_av_f64(const double* a, long long lda, long long m, int n, const double* w,
                          double* u, long long ldu, const DevStatus* status, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  if (n <= 32) return launch_av_t<double, 32, 4, 4>(a, lda, m, n, w, u, ldu, status, st);
  return launch_av_t<double, 64, 8, 4>(a, lda, m, n, w, u, ldu, status, st);
}

}  // namespace dev
}  // namespace mpsvd
