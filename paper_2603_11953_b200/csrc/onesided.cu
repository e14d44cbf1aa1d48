// The two other spectral branches of mp_thin_svd,
// proj/src/thinsvd.cpp:37-47,90-104:
//   GramCholSvd          R = chol(M) in binary64 (dense.cpp:39-58), cast to
//                        binary32 (dense.cpp:163-176), one-sided Jacobi SVD
//                        of R in binary32; sigma = sigma(R), V = V(R).
//   OneSidedJacobiOnGram one-sided Jacobi SVD of M itself in binary64;
//                        sigma = fl32(sqrt(sigma(M))), V = V(M).
// Both then share the two-sided path's epilogue (sort / sign / W = V/sigma,
// jacobi.cu finish_columns) and K7.
//
// K8 chol_upper: right-looking Cholesky in one CTA. Entry (k, j) receives
// its updates r_ik r_ij in the order i = 0, 1, ..., k-1, each product and
// difference rounded on its own (-fmad=false), then the division by r_kk:
// the same operation sequence as the reference's up-looking loop, so for
// equal M the factor is bit-identical to the reference's. The trailing
// matrix lives in shared memory when it fits, else in global memory (L2).
//
// K9 onesided_jacobi<T>: parallel round-robin one-sided Jacobi, one warp per
// column pair (the same rr_pair schedule as the two-sided solver). Per pair:
// a = |x_p|^2, b = |x_q|^2, c = x_p . x_q (lane partials with fma over rows
// lane, lane + 32, ..., then a fixed xor butterfly: every lane ends with the
// same bits), stop test |c| <= tol sqrt(a) sqrt(b) (jacobi.cpp:82-89), the
// rotation of jacobi.cpp:34-40 in the closed form the two-sided solver uses,
// and the column updates of X and V (jacobi.cpp:92-103) with one fma each.
// Converged after a sweep without rotations; ZeroColumn on a == 0 / b == 0
// (checked at the end of the sweep), NoConvergence after max_sweeps with the
// last sweep's worst |c| / sqrt(a b) (jacobi.cpp:106-108). sigma_j is the
// 2-norm of column j (max-scaled, two passes). X and V are shared-memory
// resident for small n (one CTA, __syncthreads per round), else in global
// memory with L2 loads and a cooperative grid barrier per round.
// oracle/mpsvd_port.c restates both kernels operation for operation.
#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace mpsvd {
namespace dev {

namespace {
template <typename T>
struct OsTraits;
template <>
struct OsTraits<double> {
  static __device__ __forceinline__ double sq(double x) { return sqrt(x); }
  static __device__ __forceinline__ double fm(double a, double b, double c) { return fma(a, b, c); }
  static __device__ __forceinline__ double ab(double x) { return fabs(x); }
  static __device__ __forceinline__ double mx(double a, double b) { return fmax(a, b); }
  static constexpr double kBig = 0x1p500, kSmall = 0x1p-500;
  static __device__ __forceinline__ double scl(double x, int e) { return ldexp(x, e); }
  static __device__ __forceinline__ int ex(double x) {
    int e;
    frexp(x, &e);
    return e;
  }
  static __device__ __forceinline__ double ldg(const double* p) { return __ldcg(p); }
  static __device__ __forceinline__ double cosine(double den, double rr, double) { return sqrt(den / (2.0 * rr)); }
};
template <>
struct OsTraits<float> {
  static __device__ __forceinline__ float sq(float x) { return sqrtf(x); }
  static __device__ __forceinline__ float fm(float a, float b, float c) { return fmaf(a, b, c); }
  static __device__ __forceinline__ float ab(float x) { return fabsf(x); }
  static __device__ __forceinline__ float mx(float a, float b) { return fmaxf(a, b); }
  static constexpr float kBig = 0x1p60f, kSmall = 0x1p-60f;
  static __device__ __forceinline__ float scl(float x, int e) { return ldexpf(x, e); }
  static __device__ __forceinline__ int ex(float x) {
    int e;
    frexpf(x, &e);
    return e;
  }
  static __device__ __forceinline__ float ldg(const float* p) { return __ldcg(p); }
  // cs = 1 / hypot(1, t) as the reference computes it in binary32
  // (jacobi.cpp:37): glibc's hypotf evaluates sqrt(t*t + 1) in binary64 and
  // rounds once; t*t is exact there. The closed form sqrt((|x| + r) / 2r)
  // in binary32 left V 4-5x less orthogonal than the reference's.
  static __device__ __forceinline__ float cosine(float, float, float t) {
    return 1.0f / (float)sqrt(__dadd_rn(__dmul_rn((double)t, (double)t), 1.0));
  }
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = OsTraits<T>::mx(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
}  // namespace

// ---------------------------------------------------------------------------
// K8: R = chol(M) (upper, column-major, strict lower part zero), then the
// binary32 image of R with the reference cast's checks. n x n fp64 M.
template <bool kSmem>
__global__ void __launch_bounds__(1024, 1)
chol_upper(const double* __restrict__ m_in, int n, double* __restrict__ r_glob, float* __restrict__ r32,
           DevStatus* __restrict__ status) {
  extern __shared__ double csm[];
  double* t = kSmem ? csm : r_glob;
  const int tid = threadIdx.x, bs = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = bs >> 5;
  const long long nn = (long long)n * n;
  for (long long e = tid; e < nn; e += bs) t[e] = m_in[e];
  __syncthreads();
  for (int i = 0; i < n; ++i) {
    const double d = t[(long long)i * n + i];
    if (!(d > 0.0)) {  // dense.cpp:46-47 (uniform across the block)
      if (tid == 0) {
        status->status = kNotPositiveDefinite;
        status->index = i + 1;
        status->value = d;
      }
      return;
    }
    const double rii = sqrt(d);
    __syncthreads();  // every thread has read t(i, i)
    for (int j = i + 1 + tid; j < n; j += bs) t[(long long)j * n + i] = t[(long long)j * n + i] / rii;
    if (tid == 0) t[(long long)i * n + i] = rii;
    __syncthreads();
    // trailing update t(k, j) -= r_ik r_ij, i < k <= j
    for (int j = i + 1 + warp; j < n; j += nw) {
      const double rij = t[(long long)j * n + i];
      for (int k = i + 1 + lane; k <= j; k += 32) {
        const double rik = t[(long long)k * n + i];
        const double p = rik * rij;
        t[(long long)j * n + k] = t[(long long)j * n + k] - p;
      }
    }
    __syncthreads();
  }
  // R in binary64 to r_glob (strict lower triangle zero) and its binary32
  // image with the reference cast's checks (dense.cpp:163-176): the first
  // offending entry in column-major order is reported
  __shared__ unsigned long long s_bad;
  if (tid == 0) s_bad = (unsigned long long)nn;
  __syncthreads();
  for (long long e = tid; e < nn; e += bs) {
    const int i = (int)(e % n), j = (int)(e / n);
    const double v = i <= j ? t[e] : 0.0;
    if (!isfinite(v) || fabs(v) > (double)FLT_MAX) atomicMin(&s_bad, (unsigned long long)e);
    r32[e] = (float)v;
    r_glob[e] = v;
  }
  __syncthreads();
  if (tid == 0 && s_bad < (unsigned long long)nn) {
    const double v = r_glob[s_bad];
    status->status = isfinite(v) ? kCastOverflow : kInvalid;
    status->index = (long long)(s_bad % n) + 1;  // row
    status->sweeps = (int)(s_bad / n) + 1;       // column (no sweep has run)
    status->value = v;
  }
}

// ---------------------------------------------------------------------------
// K9: one-sided Jacobi. x: m x n (column-major, ld m), v: n x n (written as
// the identity first); both of type T. Outputs: sig_raw[j] = |x_j| (as
// double), v_out = V in binary64 (unsorted; finish_columns sorts and signs).
// aux: 3 * (max_sweeps + 1) words of zeroed scratch for the grid variant.
template <typename T, bool kSmem>
__global__ void __launch_bounds__(1024, 1)
onesided_jacobi(T* __restrict__ xg, T* __restrict__ vg, int m, int n, double tol, int max_sweeps,
                DevStatus* __restrict__ status, double* __restrict__ sig_raw, double* __restrict__ v_out,
                unsigned long long* __restrict__ aux) {
  using TR = OsTraits<T>;
  extern __shared__ __align__(16) unsigned char osm[];
  T* x = kSmem ? reinterpret_cast<T*>(osm) : xg;
  T* v = kSmem ? x + (long long)m * n : vg;
  const int tid = threadIdx.x, lane = tid & 31;
  const int gwarp = (blockIdx.x * blockDim.x + tid) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int N = n + (n & 1), np = N / 2, R = N - 1;
  const T reltol = (T)tol;
  __shared__ int s_rot, s_bad;
  __shared__ unsigned long long s_worst;
  auto gsync = [&]() {
    if (kSmem)
      __syncthreads();
    else
      cg::this_grid().sync();
  };
  auto LD = [&](const T* p) -> T { return kSmem ? *p : TR::ldg(p); };
  if (status->status != kOk) return;  // an earlier stage failed (uniform)

  if (kSmem)
    for (long long e = tid; e < (long long)m * n; e += blockDim.x) x[e] = xg[e];
  for (long long e = (long long)blockIdx.x * blockDim.x + tid; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x)
    v[e] = (e % n == e / n) ? T(1) : T(0);
  gsync();

  int sweep = 0;
  bool converged = false;
  long long rotations = 0;
  for (; sweep < max_sweeps; ++sweep) {
    bool rot_any = false;
    int bad = 0x7fffffff;
    double worst = 0.0;
    for (int r = 0; r < R; ++r) {
      for (int k = gwarp; k < np; k += nwarps) {
        int p, q;
        rr_pair(n, r, k, p, q);
        if (q >= n) continue;  // bye of an odd n
        T* xp = x + (long long)p * m;
        T* xq = x + (long long)q * m;
        T a = T(0), b = T(0), c = T(0);
        for (int e = lane; e < m; e += 32) {
          const T u = LD(xp + e), w = LD(xq + e);
          a = TR::fm(u, u, a);
          b = TR::fm(w, w, b);
          c = TR::fm(u, w, c);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        c = warp_sum(c);
        if (a == T(0) || b == T(0)) {  // jacobi.cpp:80-81
          bad = min(bad, a == T(0) ? p : q);
          continue;
        }
        const T thresh = reltol * TR::sq(a) * TR::sq(b);
        worst = fmax(worst, (double)TR::ab(c) / (sqrt((double)a) * sqrt((double)b)));
        if (TR::ab(c) <= thresh) continue;
        // rotation (jacobi.cpp:34-40): x = b - a, y = 2c, r = hypot(x, y),
        // t = sign(x) y / (|x| + r) (t = 1 at x == 0), cs = sqrt((|x| + r) / 2r)
        // (binary64) or 1 / fl32(sqrt(t^2 + 1)) (binary32, see OsTraits)
        const T dx = b - a, dy = T(2) * c, ax = TR::ab(dx);
        const T big = TR::mx(ax, TR::ab(dy));
        T rr;
        if (big < TR::kBig && big > TR::kSmall) {
          rr = TR::sq(TR::fm(dx, dx, dy * dy));
        } else {
          const int e2 = TR::ex(big);
          const T xs = TR::scl(dx, -e2), ys = TR::scl(dy, -e2);
          rr = TR::scl(TR::sq(TR::fm(xs, xs, ys * ys)), e2);
        }
        const T den = ax + rr;
        const T tt = dx == T(0) ? T(1) : (dx > T(0) ? dy : -dy) / den;
        const T cs = TR::cosine(den, rr, tt);
        const T sn = cs * tt;
        for (int e = lane; e < m; e += 32) {
          const T u = LD(xp + e), w = LD(xq + e);
          xp[e] = TR::fm(cs, u, -(sn * w));
          xq[e] = TR::fm(sn, u, cs * w);
        }
        T* vp = v + (long long)p * n;
        T* vq = v + (long long)q * n;
        for (int e = lane; e < n; e += 32) {
          const T u = LD(vp + e), w = LD(vq + e);
          vp[e] = TR::fm(cs, u, -(sn * w));
          vq[e] = TR::fm(sn, u, cs * w);
        }
        rot_any = true;
        ++rotations;
      }
      if (r + 1 < R) gsync();
    }
    // end of sweep: combine the flags of every warp
    if (kSmem) {
      if (tid == 0) {
        s_rot = 0;
        s_bad = 0x7fffffff;
        s_worst = 0;
      }
      __syncthreads();
      if (lane == 0) {
        if (rot_any) atomicOr(&s_rot, 1);
        if (bad != 0x7fffffff) atomicMin(&s_bad, bad);
        atomicMax(&s_worst, (unsigned long long)__double_as_longlong(worst));
      }
      __syncthreads();
      rot_any = s_rot != 0;
      bad = s_bad;
      worst = __longlong_as_double((long long)s_worst);
      __syncthreads();
    } else {
      unsigned long long* slot = aux + 3 * sweep;
      if (lane == 0) {
        if (rot_any) atomicOr(slot + 0, 1ull);
        if (bad != 0x7fffffff) atomicMax(slot + 1, (unsigned long long)(n - bad));  // 0: none
        atomicMax(slot + 2, (unsigned long long)__double_as_longlong(worst));
      }
      cg::this_grid().sync();
      rot_any = __ldcg(slot + 0) != 0;
      const unsigned long long b1 = __ldcg(slot + 1);
      bad = b1 == 0 ? 0x7fffffff : n - (int)b1;
      worst = __longlong_as_double((long long)__ldcg(slot + 2));
    }
    if (bad != 0x7fffffff) {
      if (blockIdx.x == 0 && tid == 0) {
        status->status = kZeroColumn;
        status->index = bad + 1;
        status->value = 0.0;
        status->sweeps = sweep + 1;
      }
      return;
    }
    if (!rot_any) {
      converged = true;
      ++sweep;
      break;
    }
    if (sweep + 1 == max_sweeps && blockIdx.x == 0 && tid == 0) status->value = worst;
  }
  if (lane == 0 && rotations) atomicAdd((unsigned long long*)&status->rotations, (unsigned long long)rotations);
  if (blockIdx.x == 0 && tid == 0) status->sweeps = sweep;
  if (!converged) {
    if (blockIdx.x == 0 && tid == 0) status->status = kNoConvergence;
    return;
  }
  // sigma_j = |x_j| (max-scaled two-pass norm); V to binary64
  for (int j = gwarp; j < n; j += nwarps) {
    const T* xj = x + (long long)j * m;
    T s = T(0);
    for (int e = lane; e < m; e += 32) s = TR::mx(s, TR::ab(LD(xj + e)));
    s = warp_max(s);
    T ssq = T(0);
    if (s > T(0))
      for (int e = lane; e < m; e += 32) {
        const T y = LD(xj + e) / s;
        ssq = TR::fm(y, y, ssq);
      }
    ssq = warp_sum(ssq);
    const T nrm = s * TR::sq(ssq);
    if (lane == 0) sig_raw[j] = (double)nrm;
    for (int e = lane; e < n; e += 32) v_out[(long long)j * n + e] = (double)LD(v + (long long)j * n + e);
  }
}

// Sort (stable, descending sigma_raw), sigma in working precision, the tiny
// check of thinsvd.cpp:22-26. mode 0: GramCholSvd (sigma_raw already a
// binary32 value), 1: OneSidedJacobiOnGram (sigma = fl32(sqrt(sigma_raw))).
__global__ void onesided_sort(const double* __restrict__ sig_raw, int n, int mode, DevStatus* __restrict__ status,
                              int* __restrict__ perm, double* __restrict__ sigma) {
  __shared__ int s_bad, s_zero;
  if (threadIdx.x == 0) s_bad = s_zero = 0x7fffffff;
  __syncthreads();
  // a column that ended at zero norm (jacobi.cpp:113-114), lowest index
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (!(sig_raw[i] > 0.0)) atomicMin(&s_zero, i);
  __syncthreads();
  if (s_zero != 0x7fffffff) {
    if (threadIdx.x == 0 && status->status == kOk) {
      status->status = kZeroColumn;
      status->index = s_zero + 1;
      status->value = 0.0;
    }
    return;
  }
  const bool ok = status->status == kOk;
  for (int i = threadIdx.x; i < n && ok; i += blockDim.x) {
    const double si = sig_raw[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double sj = sig_raw[j];
      rank += sj > si || (sj == si && j < i);
    }
    perm[rank] = i;
    const double sg = mode == 0 ? si : (double)(float)sqrt(si);
    sigma[rank] = sg;
    if (!((float)sg >= FLT_MIN)) atomicMin(&s_bad, rank);
  }
  __syncthreads();
  if (ok && threadIdx.x == 0 && s_bad != 0x7fffffff) {
    status->status = kTinySingularValue;
    status->index = s_bad + 1;
    status->value = sigma[s_bad];
  }
}

size_t onesided_aux_words(int max_sweeps) { return 3 * (size_t)(max_sweeps + 1); }

cudaError_t launch_chol_upper(const double* m, int n, double* r64, float* r32, DevStatus* status, cudaStream_t st) {
  const size_t smem = (size_t)n * n * sizeof(double);
  int dev = 0, limit = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int threads = n >= 32 ? 1024 : 32 * n;  // one warp per trailing column
  if (smem <= (size_t)limit) {
    cudaFuncSetAttribute(chol_upper<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    chol_upper<true><<<1, threads, smem, st>>>(m, n, r64, r32, status);
  } else {
    chol_upper<false><<<1, threads, 0, st>>>(m, n, r64, r32, status);
  }
  return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_os(T* x, T* v, int m, int n, double tol, int max_sweeps, DevStatus* status,
                             double* sig_raw, double* v_out, unsigned long long* aux, int sm_count,
                             cudaStream_t st) {
  const int np = (n + (n & 1)) / 2;
  const size_t smem = ((size_t)m * n + (size_t)n * n) * sizeof(T);
  int dev = 0, limit = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (smem <= (size_t)limit) {
    int threads = 32 * np;
    if (threads > 1024) threads = 1024;
    if (threads < 64) threads = 64;
    auto k = onesided_jacobi<T, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<1, threads, smem, st>>>(x, v, m, n, tol, max_sweeps, status, sig_raw, v_out, aux);
    return cudaGetLastError();
  }
  cudaError_t e = cudaMemsetAsync(aux, 0, onesided_aux_words(max_sweeps) * 8, st);
  if (e != cudaSuccess) return e;
  auto k = onesided_jacobi<T, false>;
  const int threads = 512;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, 0);
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  long long grid = (np + 15) / 16;
  if (grid > (long long)sm_count * per_sm) grid = (long long)sm_count * per_sm;
  if (grid < 1) grid = 1;
  void* args[] = {&x, &v, &m, &n, &tol, &max_sweeps, &status, &sig_raw, &v_out, &aux};
  return cudaLaunchCooperativeKernel((const void*)k, dim3((unsigned)grid), dim3(threads), args, 0, st);
}

cudaError_t launch_onesided(bool f32, void* x, void* v, int m, int n, double tol, int max_sweeps, DevStatus* status,
                            double* sig_raw, double* v_out, unsigned long long* aux, int sm_count, cudaStream_t st) {
  if (f32)
    return launch_os<float>((float*)x, (float*)v, m, n, tol, max_sweeps, status, sig_raw, v_out, aux, sm_count, st);
  return launch_os<double>((double*)x, (double*)v, m, n, tol, max_sweeps, status, sig_raw, v_out, aux, sm_count, st);
}

cudaError_t launch_onesided_sort(const double* sig_raw, int n, int mode, DevStatus* status, int* perm, double* sigma,
                                 cudaStream_t st) {
  const int threads = n < 1024 ? ((n + 31) / 32) * 32 : 1024;
  onesided_sort<<<1, threads, 0, st>>>(sig_raw, n, mode, status, perm, sigma);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace mpsvd
