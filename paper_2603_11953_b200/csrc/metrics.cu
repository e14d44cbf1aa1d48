// At-scale validation metric: the row-wise backward error
// of a thin SVD, proj/src/metrics.cpp:40-70 —
//     max_i ||(U diag(sigma) V^T - A)(i, :)||_2 / ||A(i, :)||_2
// with rows of A of zero norm skipped and counted. In binary64 like the
// reference (U and V widened exactly, W = U_h diag(sigma) rounded first, then
// P = W V_h^T); the product runs on the DMMA pipe and never materialises P:
// each 128 x 64 output tile reduces its residual and row norms to per-row
// partial sums, a second kernel adds the partials of a row in column-tile
// order and takes the maximum (order-independent, so the result is
// deterministic).
#include "common.cuh"
#include "kernels.h"

namespace mpsvd {
namespace dev {
namespace bw {
constexpr int BM = 128, BN = 64, BK = 16;
constexpr int LDA_S = BM + 4, LDB_S = BN + 4;
constexpr int kStage = BK * (LDA_S + LDB_S);
}  // namespace bw

__device__ __forceinline__ void dmma884_bw(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// T: float (working) or double (higher) storage of A, U, V (column-major).
// partial[(ct * m + row) * 2 + {0: residual^2, 1: |A row|^2}] over the tile's columns.
template <typename T>
__global__ void __launch_bounds__(256, 2)
backward_tile(const T* __restrict__ a, long long lda, const T* __restrict__ u, long long ldu,
              const double* __restrict__ sigma, const T* __restrict__ v, long long ldv, long long m, int n,
              double* __restrict__ partial) {
  using namespace bw;
  extern __shared__ double sm[];  // 2 stages; reused for the row reduction
  auto red = reinterpret_cast<double(*)[2][2]>(sm);  // [row][column half][res, row]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wi = warp >> 1, wj = warp & 1, g = lane >> 2, t = lane & 3;
  const long long r0 = (long long)blockIdx.x * BM;
  const int c0 = blockIdx.y * BN;

  auto stage = [&](int ch, int buf) {
    double* as = sm + buf * kStage;
    double* bs = as + BK * LDA_S;
    const int k0 = ch * BK;
    // W(i, l) = U_h(i, l) * sigma_l  (the reference's scale_columns, rounded)
    for (int e = tid; e < BK * BM; e += 256) {
      const int kk = e / BM, i = e - kk * BM;
      const long long row = r0 + i;
      const int l = k0 + kk;
      as[kk * LDA_S + i] = (l < n && row < m) ? (double)u[(long long)l * ldu + row] * sigma[l] : 0.0;
    }
    // B(l, j) = V_h(j, l)
    for (int e = tid; e < BK * BN; e += 256) {
      const int kk = e / BN, jj = e - kk * BN;
      const int l = k0 + kk, col = c0 + jj;
      bs[kk * LDB_S + jj] = (l < n && col < n) ? (double)v[(long long)l * ldv + col] : 0.0;
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nch = (n + BK - 1) / BK;
  stage(0, 0);
  __syncthreads();
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) stage(ch + 1, (ch + 1) & 1);
    const double* as = sm + (ch & 1) * kStage;
    const double* bs = as + BK * LDA_S;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = as[(kk + t) * LDA_S + 32 * wi + 8 * i + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = bs[(kk + t) * LDB_S + 32 * wj + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884_bw(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
    __syncthreads();
  }
  // residual and row norm of this thread's 2 x 4 x 2 entries per row group;
  // reduced over the 4 lanes sharing a row (t), then over the two column
  // halves (wj) in shared memory
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int lr = 32 * wi + 8 * i + g;
    const long long row = r0 + lr;
    double res = 0.0, rs = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = c0 + 32 * wj + 8 * j + 2 * t + h;
        if (row < m && col < n) {
          const double x = (double)a[(long long)col * lda + row];
          const double d = acc[i][j][h] - x;
          res = fma(d, d, res);
          rs = fma(x, x, rs);
        }
      }
    res += __shfl_xor_sync(0xffffffffu, res, 1);
    rs += __shfl_xor_sync(0xffffffffu, rs, 1);
    res += __shfl_xor_sync(0xffffffffu, res, 2);
    rs += __shfl_xor_sync(0xffffffffu, rs, 2);
    if (t == 0) {
      red[lr][wj][0] = res;
      red[lr][wj][1] = rs;
    }
  }
  __syncthreads();
  if (tid < BM && r0 + tid < m) {
    const long long row = r0 + tid;
    partial[((long long)blockIdx.y * m + row) * 2 + 0] = red[tid][0][0] + red[tid][1][0];
    partial[((long long)blockIdx.y * m + row) * 2 + 1] = red[tid][0][1] + red[tid][1][1];
  }
}

// out[0] = max relative residual (as uint64 bits of a non-negative double),
// out[1] = number of zero rows
__global__ void backward_reduce(const double* __restrict__ partial, long long m, int ntiles,
                                unsigned long long* __restrict__ out) {
  double worst = 0.0;
  unsigned long long skipped = 0;
  for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < m;
       row += (long long)gridDim.x * blockDim.x) {
    double res = 0.0, rs = 0.0;
    for (int ct = 0; ct < ntiles; ++ct) {
      res += partial[((long long)ct * m + row) * 2 + 0];
      rs += partial[((long long)ct * m + row) * 2 + 1];
    }
    if (rs == 0.0) {
      ++skipped;
      continue;
    }
    worst = fmax(worst, sqrt(res) / sqrt(rs));
  }
  for (int o = 16; o > 0; o >>= 1) {
    worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    skipped += __shfl_xor_sync(0xffffffffu, skipped, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out[0], (unsigned long long)__double_as_longlong(worst));  // ordered for doubles >= 0
    atomicAdd(&out[1], skipped);
  }
}

template <typename T>
static cudaError_t backward_t(const T* a, long long lda, const T* u, long long ldu, const double* sigma, const T* v,
                              long long ldv, long long m, int n, double* partial, unsigned long long* out,
                              cudaStream_t st) {
  using namespace bw;
  cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), st);
  if (e != cudaSuccess || m <= 0) return e;
  const dim3 grid((unsigned)((m + BM - 1) / BM), (unsigned)((n + BN - 1) / BN));
  const int smem = 2 * kStage * (int)sizeof(double);
  e = cudaFuncSetAttribute(backward_tile<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  backward_tile<T><<<grid, 256, smem, st>>>(a, lda, u, ldu, sigma, v, ldv, m, n, partial);
  long long rb = (m + 255) / 256;
  if (rb > 4 * 148) rb = 4 * 148;
  backward_reduce<<<(unsigned)rb, 256, 0, st>>>(partial, m, (int)grid.y, out);
  return cudaGetLastError();
}

size_t backward_partial_elems(long long m, int n) { return (size_t)m * ((n + bw::BN - 1) / bw::BN) * 2; }

cudaError_t launch_backward_error(bool f64, const void* a, long long lda, const void* u, long long ldu,
                                  const double* sigma, const void* v, long long ldv, long long m, int n,
                                  double* partial, unsigned long long* out, cudaStream_t st) {
  if (f64)
    return backward_t<double>((const double*)a, lda, (const double*)u, ldu, sigma, (const double*)v, ldv, m, n,
                              partial, out, st);
  return backward_t<float>((const float*)a, lda, (const float*)u, ldu, sigma, (const float*)v, ldv, m, n, partial,
                           out, st);
}

}  // namespace dev
}  // namespace mpsvd
