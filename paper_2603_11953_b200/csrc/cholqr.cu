// K10: the row-wise forward substitution of the mixed-precision Cholesky QR
// (proj/src/thinsvd.cpp:125-154):
//     Q(i,:) R = A(i,:)  for every row i, in binary32,
// with R = fl32(chol(A^T A)) from K1 + K8. Every row is independent, so one
// thread owns one row: q_j = (a_ij - q_0 r_0j - q_1 r_1j - ... - q_{j-1}
// r_{j-1,j}) / r_jj, each product and difference rounded on its own
// (-fmad=false) and a true division — the reference's operation sequence per
// entry (its loop is vectorised over rows, k ascending, then the divide), so
// for equal R the factor Q is bit-identical to the reference's.
//
// Layout: the solved prefix of the thread's row lives in shared memory
// (pitch p with p = 4 mod 32 words, so the 8 threads of a 128-bit access
// phase hit distinct bank quads); R is read through the read-only path with
// warp-uniform addresses (one broadcast transaction per load); A is read and
// Q written column by column, coalesced across the rows of a CTA. The loop
// is bound by the FP32 pipe (one multiply + one subtract per (j, k)), not by
// HBM (A and Q each cross it once).
#include "common.cuh"
#include "kernels.h"

namespace mpsvd {
namespace dev {

constexpr int kCqJ = 4;  // columns solved together (independent chains per thread)
__host__ __device__ __forceinline__ int cholqr_ld(int n) { return (n + kCqJ - 1) / kCqJ * kCqJ; }
__host__ __device__ __forceinline__ int cholqr_pitch(int n) {
  int p = cholqr_ld(n);
  p += ((4 - p % 32) + 32) % 32;
  return p;
}

// kRs: R staged in shared memory as an ldr x ldr column-major block (ldr =
// n rounded up to kCqJ, zero padded), and the row solved kCqJ columns at a time:
// for a column block J = [j0, j0 + kCqJ) the prefix k < j0 is applied as 4 x kCqJ
// tiles (one float4 of the row's q, kCqJ float4 broadcasts of R), every s_j
// still taking its k in ascending order; then the block's triangle and the
// divisions. Else (R too large for shared memory) one column at a time with
// R through the read-only path. The row of A is staged first (all n loads in
// flight at once), then solved in place.
__global__ void __launch_bounds__(256)
cholqr_rows_rs(const float* __restrict__ a, long long lda, long long m, int n, const float* __restrict__ r,
               float* __restrict__ q, long long ldq, const DevStatus* __restrict__ status) {
  if (status->status != kOk) return;
  extern __shared__ __align__(16) float cq_smem[];
  const int p = cholqr_pitch(n), ldr = cholqr_ld(n);
  float* rs = cq_smem;
  float* qs = cq_smem + (size_t)ldr * ldr + (size_t)threadIdx.x * p;
  for (int e = threadIdx.x; e < ldr * ldr; e += blockDim.x) {
    const int i = e % ldr, j = e / ldr;
    rs[e] = (i < n && j < n) ? r[(size_t)j * n + i] : 0.0f;
  }
  __syncthreads();
  for (long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (long long)gridDim.x * blockDim.x) {
    for (int j = 0; j < n; ++j) qs[j] = a[(size_t)j * lda + row];
    for (int j0 = 0; j0 < n; j0 += kCqJ) {
      float sj[kCqJ];
#pragma unroll
      for (int h = 0; h < kCqJ; h += 4) {
        const float4 sv = *reinterpret_cast<const float4*>(qs + j0 + h);
        sj[h] = sv.x;
        sj[h + 1] = sv.y;
        sj[h + 2] = sv.z;
        sj[h + 3] = sv.w;
      }
      const float* r0 = rs + (size_t)j0 * ldr;
      for (int k = 0; k < j0; k += 4) {
        const float4 qv = *reinterpret_cast<const float4*>(qs + k);
#pragma unroll
        for (int jj = 0; jj < kCqJ; ++jj) {
          const float4 rv = *reinterpret_cast<const float4*>(r0 + (size_t)jj * ldr + k);
          sj[jj] = sj[jj] - qv.x * rv.x;
          sj[jj] = sj[jj] - qv.y * rv.y;
          sj[jj] = sj[jj] - qv.z * rv.z;
          sj[jj] = sj[jj] - qv.w * rv.w;
        }
      }
#pragma unroll
      for (int jj = 0; jj < kCqJ; ++jj) {
        if (j0 + jj < n) {
          const float* rj = r0 + (size_t)jj * ldr;
#pragma unroll
          for (int kk = 0; kk < jj; ++kk) sj[jj] = sj[jj] - sj[kk] * rj[j0 + kk];
          sj[jj] = sj[jj] / rj[j0 + jj];
          q[(size_t)(j0 + jj) * ldq + row] = sj[jj];
        }
      }
#pragma unroll
      for (int h = 0; h < kCqJ; h += 4)
        *reinterpret_cast<float4*>(qs + j0 + h) = make_float4(sj[h], sj[h + 1], sj[h + 2], sj[h + 3]);
    }
  }
}

// R read through the read-only path (R too large for shared memory).
__global__ void __launch_bounds__(256)
cholqr_rows_ldg(const float* __restrict__ a, long long lda, long long m, int n, const float* __restrict__ r,
                float* __restrict__ q, long long ldq, const DevStatus* __restrict__ status) {
  if (status->status != kOk) return;
  extern __shared__ __align__(16) float cq_smem[];
  float* qs = cq_smem + (size_t)threadIdx.x * cholqr_pitch(n);
  for (long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (long long)gridDim.x * blockDim.x) {
    for (int j = 0; j < n; ++j) qs[j] = a[(size_t)j * lda + row];
    for (int j = 0; j < n; ++j) {
      float s = qs[j];
      const float* rj = r + (size_t)j * n;
      int k = 0;
      for (; k + 4 <= j; k += 4) {
        const float4 qv = *reinterpret_cast<const float4*>(qs + k);
        s = s - qv.x * __ldg(rj + k);
        s = s - qv.y * __ldg(rj + k + 1);
        s = s - qv.z * __ldg(rj + k + 2);
        s = s - qv.w * __ldg(rj + k + 3);
      }
      for (; k < j; ++k) s = s - qs[k] * __ldg(rj + k);
      s = s / __ldg(rj + j);
      qs[j] = s;
      q[(size_t)j * ldq + row] = s;
    }
  }
}

cudaError_t launch_cholqr_rows(const float* a, long long lda, long long m, int n, const float* r, float* q,
                               long long ldq, const DevStatus* status, int sm_count, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  const size_t per_row = (size_t)cholqr_pitch(n) * sizeof(float);
  const size_t r_bytes = (size_t)cholqr_ld(n) * cholqr_ld(n) * sizeof(float);
  const size_t budget = 200 * 1024;
  const void* k;
  int threads;
  size_t smem;
  if (r_bytes + 64 * per_row <= budget) {
    threads = (int)((budget - r_bytes) / per_row) / 32 * 32;
    if (threads > 256) threads = 256;
    smem = r_bytes + (size_t)threads * per_row;
    k = (const void*)cholqr_rows_rs;
  } else {
    threads = (int)(budget / per_row) / 32 * 32;
    if (threads > 256) threads = 256;
    if (threads < 32) threads = 32;
    smem = (size_t)threads * per_row;
    k = (const void*)cholqr_rows_ldg;
  }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
  if (per_sm < 1) per_sm = 1;
  long long grid = (m + threads - 1) / threads;
  if (grid > (long long)sm_count * per_sm) grid = (long long)sm_count * per_sm;
  void* args[] = {&a, &lda, &m, &n, &r, &q, &ldq, &status};
  return cudaLaunchKernel(k, dim3((unsigned)grid), dim3(threads), args, smem, st);
}

}  // namespace dev
}  // namespace mpsvd
