// K7: U = A * (V Sigma^-1) in working precision.
//
// Reference semantics: matmul(a, scale_columns(v, sigma, invert))
// (proj/src/thinsvd.cpp:110-113, proj/src/dense.cpp:83-96,214-232): W is
// formed first (true division, done by finish_columns in jacobi.cu and stored
// row-major "W^T" with a 16-byte aligned leading dimension), then every U
// entry accumulates A(i,l)*W(l,j) over ascending l. Here each entry is one
// fma chain over ascending l (the reference's x86 build rounds the product
// and the sum separately; same order).
//
// Tiling: a CTA owns BM rows x NB output columns (NB >= n for n <= 128, so A
// is streamed from HBM exactly once and U written once); A and W^T slices of
// BK columns are staged into shared memory by cp.async (16-byte LDGSTS,
// zero-filled at the matrix edges) in a two-stage pipeline; each thread keeps
// a TM x TN register tile and reads its operands with 128-bit shared loads.
#include "common.cuh"
#include "kernels.h"

namespace mpsvd {
namespace dev {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <typename T, int NB, int TM, int TN, int BK>
struct AvShape {
  static constexpr int CG = NB / TN;  // column groups
  static constexpr int RG = 256 / CG; // row groups
  static constexpr int BM = RG * TM;  // rows per CTA
  static constexpr int V = 16 / sizeof(T);
  static constexpr size_t smem = 2 * (size_t)BK * (BM + NB) * sizeof(T);
};

// kAsync: 16-byte cp.async staging (needs lda % V == 0 and a 16-byte aligned A).
template <typename T, int NB, int TM, int TN, int BK, bool kAsync>
__global__ void __launch_bounds__(256)
av_kernel(const T* __restrict__ a, long long lda, long long m, int n, const T* __restrict__ wt, int ldw,
          T* __restrict__ u, long long ldu, const DevStatus* __restrict__ status) {
  using S = AvShape<T, NB, TM, TN, BK>;
  constexpr int BM = S::BM, V = S::V;
  if (status && status->status != kOk) return;
  extern __shared__ __align__(16) unsigned char avsm[];
  T* as = reinterpret_cast<T*>(avsm);  // [2][BK][BM]
  T* ws = as + 2 * BK * BM;            // [2][BK][NB]
  const int tid = threadIdx.x;
  const int tx = tid % S::CG, ty = tid / S::CG;
  const long long r0 = (long long)blockIdx.x * BM;
  const int c0 = blockIdx.y * NB;

  auto issue = [&](int l0, int buf) {
    T* ad = as + buf * BK * BM;
    T* wd = ws + buf * BK * NB;
    if (kAsync) {
      constexpr int AV = BK * BM / V;  // 16-byte vectors of the A slice
      for (int e = tid; e < AV; e += 256) {
        const int kk = e / (BM / V), iv = e - kk * (BM / V);
        const long long row = r0 + (long long)iv * V;
        const int l = l0 + kk;
        long long rem = (m - row) * (long long)sizeof(T);
        int bytes = (l < n && rem > 0) ? (rem >= 16 ? 16 : (int)rem) : 0;
        const T* src = bytes ? a + (long long)l * lda + row : a;
        cp_async16(ad + kk * BM + iv * V, src, bytes);
      }
    } else {
      for (int e = tid; e < BK * BM; e += 256) {
        const int kk = e / BM, i = e - kk * BM;
        const long long row = r0 + i;
        const int l = l0 + kk;
        ad[kk * BM + i] = (l < n && row < m) ? a[(long long)l * lda + row] : T(0);
      }
    }
    constexpr int WV = BK * NB / V;
    for (int e = tid; e < WV; e += 256) {
      const int kk = e / (NB / V), jv = e - kk * (NB / V);
      const int l = l0 + kk, col = c0 + jv * V;
      const int rem = (n - col) * (int)sizeof(T);
      const int bytes = (l < n && rem > 0) ? (rem >= 16 ? 16 : rem) : 0;
      const T* src = bytes ? wt + (long long)l * ldw + col : wt;
      cp_async16(wd + kk * NB + jv * V, src, bytes);
    }
    cp_async_commit();
  };

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  const int nchunks = (n + BK - 1) / BK;
  issue(0, 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int cur = ch & 1;
    if (ch + 1 < nchunks) {
      issue((ch + 1) * BK, cur ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const T* ac = as + cur * BK * BM + ty * TM;
    const T* wc = ws + cur * BK * NB + tx * TN;
    const int kmax = min(BK, n - ch * BK);
#pragma unroll 4
    for (int k = 0; k < kmax; ++k) {
      T av[TM], wv[TN];
#pragma unroll
      for (int i = 0; i < TM; i += V) *reinterpret_cast<float4*>(&av[i]) = *reinterpret_cast<const float4*>(ac + k * BM + i);
#pragma unroll
      for (int j = 0; j < TN; j += V) *reinterpret_cast<float4*>(&wv[j]) = *reinterpret_cast<const float4*>(wc + k * NB + j);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i], wv[j], acc[i][j]);
    }
    __syncthreads();
  }
  const long long rbase = r0 + (long long)ty * TM;
  const bool vec_ok = kAsync && (ldu % V == 0) && (rbase + TM <= m);
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    const int col = c0 + tx * TN + j;
    if (col >= n) continue;
    T* dst = u + (long long)col * ldu + rbase;
    if (vec_ok) {
#pragma unroll
      for (int i = 0; i < TM; i += V) {
        T tmp[V];
#pragma unroll
        for (int q = 0; q < V; ++q) tmp[q] = acc[i + q][j];
        *reinterpret_cast<float4*>(dst + i) = *reinterpret_cast<const float4*>(tmp);
      }
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
        if (rbase + i < m) dst[i] = acc[i][j];
    }
  }
}

template <typename T, int NB, int TM, int TN, int BK>
static cudaError_t launch_av_t(const T* a, long long lda, long long m, int n, const T* w, int ldw, T* u,
                               long long ldu, const DevStatus* status, cudaStream_t st) {
  using S = AvShape<T, NB, TM, TN, BK>;
  const bool async_ok = (lda % S::V == 0) && (reinterpret_cast<uintptr_t>(a) % 16 == 0);
  dim3 grid((unsigned)((m + S::BM - 1) / S::BM), (unsigned)((n + NB - 1) / NB));
  if (async_ok) {
    auto k = av_kernel<T, NB, TM, TN, BK, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::smem);
    k<<<grid, 256, S::smem, st>>>(a, lda, m, n, w, ldw, u, ldu, status);
  } else {
    auto k = av_kernel<T, NB, TM, TN, BK, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::smem);
    k<<<grid, 256, S::smem, st>>>(a, lda, m, n, w, ldw, u, ldu, status);
  }
  return cudaGetLastError();
}



cudaError_t launch_av_f32(const float* a, long long lda, long long m, int n, const float* w, float* u,
                          long long ldu, const DevStatus* status, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  const int ldw = av_ldw(n);
  if (n <= 32) return launch_av_t<float, 32, 8, 8, 16>(a, lda, m, n, w, ldw, u, ldu, status, st);
  if (n <= 64) return launch_av_t<float, 64, 8, 8, 32>(a, lda, m, n, w, ldw, u, ldu, status, st);
  return launch_av_t<float, 128, 8, 8, 32>(a, lda, m, n, w, ldw, u, ldu, status, st);
}

cudaError_t launch_av_f64(const double* a, long long lda, long long m, int n, const double* w, double* u,
                          long long ldu, const DevStatus* status, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  const int ldw = av_ldw(n);
  if (n <= 32) return launch_av_t<double, 32, 8, 4, 16>(a, lda, m, n, w, ldw, u, ldu, status, st);
  return launch_av_t<double, 64, 8, 4, 32>(a, lda, m, n, w, ldw, u, ldu, status, st);
}


// ---------------------------------------------------------------------------
// K7 (fp64) on the DMMA pipe: U = A * W, A m x n column-major, W row-major
// (wt[l * ldw + j] = W(l, j)). CTA tile 128 rows x 64 columns, K chunks of 16
// double-buffered with cp.async; 8 warps as 4 (rows) x 2 (columns), each a
// 32 x 32 block = 4 x 4 mma.sync.m8n8k4.f64 tiles. Shared tiles are k-major
// with a 4-word pad so that the fragment loads (k = t, rows 8i + g) hit 32
// distinct banks. fp64 products and sums on the tensor pipe: U differs from an
// fp64 fma chain by summation order only.
namespace av64 {
constexpr int BM = 128, BN = 64, BK = 16;
constexpr int LDA_S = BM + 4, LDW_S = BN + 4;
constexpr int kStage = BK * (LDA_S + LDW_S);  // doubles per stage
}  // namespace av64

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256, 2)
av_dmma_f64(const double* __restrict__ a, long long lda, long long m, int n, const double* __restrict__ wt, int ldw,
            double* __restrict__ u, long long ldu, const DevStatus* __restrict__ status) {
  using namespace av64;
  if (status && status->status != kOk) return;
  extern __shared__ __align__(16) double av64s[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wi = warp >> 1, wj = warp & 1, g = lane >> 2, t = lane & 3;
  const long long r0 = (long long)blockIdx.x * BM;
  const int c0 = blockIdx.y * BN;
  const bool vec_a = (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0);
  const bool vec_w = (ldw % 2 == 0) && ((reinterpret_cast<uintptr_t>(wt) & 15) == 0);

  auto stage = [&](int ch, int buf) {
    double* as = av64s + buf * kStage;
    double* ws = as + BK * LDA_S;
    const int k0 = ch * BK;
    // A: BK columns x BM rows, 16-byte pieces (2 rows)
    for (int e = tid; e < BK * BM / 2; e += 256) {
      const int kk = e / (BM / 2), ip = e - kk * (BM / 2);
      const long long row = r0 + 2 * ip;
      const int l = k0 + kk;
      double* dst = as + kk * LDA_S + 2 * ip;
      if (vec_a && l < n && row + 1 < m) {
        cp_async16(dst, a + (long long)l * lda + row, 16);
      } else {
        dst[0] = (l < n && row < m) ? a[(long long)l * lda + row] : 0.0;
        dst[1] = (l < n && row + 1 < m) ? a[(long long)l * lda + row + 1] : 0.0;
      }
    }
    // W: BK rows x BN columns
    for (int e = tid; e < BK * BN / 2; e += 256) {
      const int kk = e / (BN / 2), jp = e - kk * (BN / 2);
      const int l = k0 + kk, col = c0 + 2 * jp;
      double* dst = ws + kk * LDW_S + 2 * jp;
      if (vec_w && l < n && col + 1 < n) {
        cp_async16(dst, wt + (long long)l * ldw + col, 16);
      } else {
        dst[0] = (l < n && col < n) ? wt[(long long)l * ldw + col] : 0.0;
        dst[1] = (l < n && col + 1 < n) ? wt[(long long)l * ldw + col + 1] : 0.0;
      }
    }
    cp_async_commit();
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nch = (n + BK - 1) / BK;
  stage(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      stage(ch + 1, (ch + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = av64s + (ch & 1) * kStage;
    const double* ws = as + BK * LDA_S;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = as[(kk + t) * LDA_S + 32 * wi + 8 * i + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = ws[(kk + t) * LDW_S + 32 * wj + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long row = r0 + 32 * wi + 8 * i + g;
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = c0 + 32 * wj + 8 * j + 2 * t;
      if (col < n) u[(long long)col * ldu + row] = acc[i][j][0];
      if (col + 1 < n) u[(long long)(col + 1) * ldu + row] = acc[i][j][1];
    }
  }
}

cudaError_t launch_av_dmma_f64(const double* a, long long lda, long long m, int n, const double* w, double* u,
                               long long ldu, const DevStatus* status, cudaStream_t st) {
  using namespace av64;
  if (m <= 0) return cudaSuccess;
  const size_t smem = 2 * (size_t)kStage * sizeof(double);
  cudaFuncSetAttribute(av_dmma_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  // per device
  dim3 grid((unsigned)((m + BM - 1) / BM), (unsigned)((n + BN - 1) / BN));
  av_dmma_f64<<<grid, 256, smem, st>>>(a, lda, m, n, w, av_ldw(n), u, ldu, status);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace mpsvd
