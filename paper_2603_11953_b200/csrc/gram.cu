// K1 / K2: the higher-precision Gram product M = A^T A.
//
// Reference semantics: partitioned_gram (proj/src/parallel_gram.cpp:265-298)
// on cast(A, Higher) (proj/src/thinsvd.cpp:61-70): fp32 entries widened
// exactly, fp64 products exact, fp64 accumulation; 16 logical row blocks
// (thinsvd.cpp:66) combined by a fixed binary tree (parallel_gram.cpp:93-102);
// upper triangle computed and mirrored (parallel_gram.cpp:28-29).
//
// Device layout: the n x n output is cut into 64x64 tiles;
// only upper tile pairs (I <= J) are computed. Every logical block is split
// into a fixed number of row ranges ("splits"), one CTA per (tile pair,
// split). Each CTA streams its rows of the <=128 columns it needs through
// shared memory in 32-row chunks (widened to fp64 once, while staging) and
// writes a 64x64 partial tile. gram_combine sums the splits of a block in
// order, then the blocks along the reference's tree, and mirrors: the result
// is run-to-run deterministic and exactly symmetric.
//
//   K1 gram_f32_dmma : fp32 input, fp64 accumulation on the DMMA tensor
//                      pipe (mma.sync.m8n8k4.f64, measured 37.0 TF on B200
//                      vs 34.2 TF for DFMA, profiles/r01_microbench.txt).
//   K2 gram_f64_dd   : fp64 input, exact products (two_prod) accumulated in
//                      double-double (Dot2: TwoSum of the high parts, plain
//                      sum of the error terms), proj/tests/support/dd.cpp:75-88.
#include "common.cuh"
#include "kernels.h"

namespace mpsvd {
namespace dev {

constexpr int kTile = 64;
constexpr int kKC = 32;        // rows per staged chunk
constexpr int kLDK = kKC + 4;  // K1: doubles per smem column; 8g+2t bank pattern

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// K1. 128 threads = 4 warps in a 2x2 grid, each warp a 32x32 block of the
// 64x64 output tile = 4x4 DMMA tiles of 8x8. smem: [2 buffers][ncol][kLDK].
__global__ void __launch_bounds__(128, 2)
gram_f32_dmma(const float* __restrict__ a, long long lda, int n, const int2* __restrict__ tiles,
              const longlong2* __restrict__ splits, double* __restrict__ partials, int ntp) {
  extern __shared__ __align__(16) double smem_k1[];
  const int tp = blockIdx.x, s = blockIdx.y;
  const int2 tij = tiles[tp];
  const bool diag = tij.x == tij.y;
  const int ncol = diag ? kTile : 2 * kTile;
  const int c0 = tij.x * kTile, c1 = tij.y * kTile;
  const long long r0 = splits[s].x, r1 = splits[s].y;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wi = warp >> 1, wj = warp & 1;
  const int g = lane >> 2, t = lane & 3;
  const bool warp_active = !(diag && wi > wj);
  const int boff = diag ? 0 : kTile;

  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 4; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;

  // Thread -> (column, row) of a chunk: warp w, iteration it loads column
  // 4*it+w, rows 0..31 -> one 128-byte segment per warp per iteration.
  const int niter = ncol / 4;  // 16 or 32
  float pre[32];
  auto load_chunk = [&](long long kr) {
#pragma unroll
    for (int it = 0; it < 32; ++it) {
      if (it < niter) {
        const int lc = it * 4 + warp;
        const int gc = lc < kTile ? c0 + lc : c1 + (lc - kTile);
        const long long row = kr + lane;
        pre[it] = (gc < n && row < r1) ? __ldg(a + (long long)gc * lda + row) : 0.0f;
      }
    }
  };
  auto store_chunk = [&](double* buf) {
#pragma unroll
    for (int it = 0; it < 32; ++it)
      if (it < niter) buf[(it * 4 + warp) * kLDK + lane] = (double)pre[it];
  };

  const long long nchunks = (r1 - r0 + kKC - 1) / kKC;
  double* buf0 = smem_k1;
  double* buf1 = smem_k1 + 2 * kTile * kLDK;
  if (nchunks > 0) {
    load_chunk(r0);
    store_chunk(buf0);
  }
  __syncthreads();
  for (long long ch = 0; ch < nchunks; ++ch) {
    double* cur = (ch & 1) ? buf1 : buf0;
    double* nxt = (ch & 1) ? buf0 : buf1;
    const bool more = ch + 1 < nchunks;
    if (more) load_chunk(r0 + (ch + 1) * kKC);
    if (warp_active) {
#pragma unroll
      for (int kk = 0; kk < kKC; kk += 4) {
        double fa[4], fb[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) fa[mi] = cur[(32 * wi + 8 * mi + g) * kLDK + kk + t];
#pragma unroll
        for (int nj = 0; nj < 4; ++nj) fb[nj] = cur[(boff + 32 * wj + 8 * nj + g) * kLDK + kk + t];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj)
            if (!diag || (32 * wi + 8 * mi) <= (32 * wj + 8 * nj))
              dmma_8x8x4(acc[mi][nj][0], acc[mi][nj][1], fa[mi], fb[nj]);
      }
    }
    if (more) store_chunk(nxt);
    __syncthreads();
  }

  // Epilogue: row-major 64x64 partial tile; entries below the diagonal of a
  // diagonal tile are never read by gram_combine.
  double* out = partials + ((long long)s * ntp + tp) * (kTile * kTile);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 4; ++nj) {
      const int r = 32 * wi + 8 * mi + g;
      const int c = 32 * wj + 8 * nj + 2 * t;
      double2 v;
      v.x = acc[mi][nj][0];
      v.y = acc[mi][nj][1];
      *reinterpret_cast<double2*>(out + r * kTile + c) = v;
    }
}

// ---------------------------------------------------------------------------
// K2. 256 threads in a 16x16 grid, each a 4x4 block of the 64x64 tile, Dot2
// accumulation. smem: [2 buffers][kKC][kLDC] (row k, columns contiguous).
constexpr int kLDC = 2 * kTile + 2;

__global__ void __launch_bounds__(256, 1)
gram_f64_dd(const double* __restrict__ a, long long lda, int n, const int2* __restrict__ tiles,
            const longlong2* __restrict__ splits, double2* __restrict__ partials, int ntp) {
  extern __shared__ __align__(16) double smem_k2[];
  const int tp = blockIdx.x, s = blockIdx.y;
  const int2 tij = tiles[tp];
  const bool diag = tij.x == tij.y;
  const int ncol = diag ? kTile : 2 * kTile;
  const int c0 = tij.x * kTile, c1 = tij.y * kTile;
  const long long r0 = splits[s].x, r1 = splits[s].y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ty = tid >> 4, tx = tid & 15;
  const int boff = diag ? 0 : kTile;
  const bool active = !diag || ty <= tx;

  double sh[4][4], sl[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) sh[u][v] = sl[u][v] = 0.0;

  const int niter = ncol / 8;  // 8 or 16 (256 threads x 16 = 32 rows x 128 cols)
  double pre[16];
  auto load_chunk = [&](long long kr) {
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      if (it < niter) {
        const int lc = it * 8 + warp;
        const int gc = lc < kTile ? c0 + lc : c1 + (lc - kTile);
        const long long row = kr + lane;
        pre[it] = (gc < n && row < r1) ? __ldg(a + (long long)gc * lda + row) : 0.0;
      }
    }
  };
  auto store_chunk = [&](double* buf) {
#pragma unroll
    for (int it = 0; it < 16; ++it)
      if (it < niter) buf[lane * kLDC + it * 8 + warp] = pre[it];
  };

  const long long nchunks = (r1 - r0 + kKC - 1) / kKC;
  double* buf0 = smem_k2;
  double* buf1 = smem_k2 + kKC * kLDC;
  if (nchunks > 0) {
    load_chunk(r0);
    store_chunk(buf0);
  }
  __syncthreads();
  for (long long ch = 0; ch < nchunks; ++ch) {
    double* cur = (ch & 1) ? buf1 : buf0;
    double* nxt = (ch & 1) ? buf0 : buf1;
    const bool more = ch + 1 < nchunks;
    if (more) load_chunk(r0 + (ch + 1) * kKC);
    if (active) {
#pragma unroll 4
      for (int k = 0; k < kKC; ++k) {
        const double2 a01 = *reinterpret_cast<const double2*>(cur + k * kLDC + 4 * ty);
        const double2 a23 = *reinterpret_cast<const double2*>(cur + k * kLDC + 4 * ty + 2);
        const double2 b01 = *reinterpret_cast<const double2*>(cur + k * kLDC + boff + 4 * tx);
        const double2 b23 = *reinterpret_cast<const double2*>(cur + k * kLDC + boff + 4 * tx + 2);
        const double av[4] = {a01.x, a01.y, a23.x, a23.y};
        const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            // Dot2: (p, e) = TwoProd(a, b); (s, sig) = TwoSum(s, p); c += e + sig
            const double p = av[u] * bv[v];
            const double e = fma(av[u], bv[v], -p);
            const double sn = sh[u][v] + p;
            const double bb = sn - sh[u][v];
            const double sig = (sh[u][v] - (sn - bb)) + (p - bb);
            sh[u][v] = sn;
            sl[u][v] += e + sig;
          }
      }
    }
    if (more) store_chunk(nxt);
    __syncthreads();
  }
  double2* out = partials + ((long long)s * ntp + tp) * (kTile * kTile);
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const dd r = quick_two_sum(sh[u][v], sl[u][v]);
      out[(4 * ty + u) * kTile + 4 * tx + v] = make_double2(r.hi, r.lo);
    }
}

// ---------------------------------------------------------------------------
// Combine, two coalesced passes:
//   gram_block_sums: for every (tile pair, tile element, logical block) the
//                    block's splits summed in ascending order;
//   gram_tree:       the reference's fixed tree over the block sums
//                    (parallel_gram.cpp:93-102), written to both triangles.
template <typename ST>
__device__ __forceinline__ ST st_add(ST a, ST b);
template <>
__device__ __forceinline__ double st_add<double>(double a, double b) { return a + b; }
template <>
__device__ __forceinline__ double2 st_add<double2>(double2 a, double2 b) {
  const dd r = dd_add(dd_make(a.x, a.y), dd_make(b.x, b.y));
  return make_double2(r.hi, r.lo);
}
template <typename ST>
__device__ __forceinline__ ST st_zero();
template <>
__device__ __forceinline__ double st_zero<double>() { return 0.0; }
template <>
__device__ __forceinline__ double2 st_zero<double2>() { return make_double2(0.0, 0.0); }

template <typename ST>
__global__ void __launch_bounds__(256)
gram_block_sums(const ST* __restrict__ partials, int ntp, const int* __restrict__ block_split_begin,
                ST* __restrict__ sums) {
  const int tp = blockIdx.x, b = blockIdx.z;
  const int e = blockIdx.y * 256 + threadIdx.x;  // tile element, 16 x 256 = 64 x 64
  const int s0 = block_split_begin[b], s1 = block_split_begin[b + 1];
  ST acc = st_zero<ST>();
  for (int sidx = s0; sidx < s1; ++sidx)
    acc = st_add<ST>(acc, partials[((long long)sidx * ntp + tp) * (kTile * kTile) + e]);
  sums[((long long)b * ntp + tp) * (kTile * kTile) + e] = acc;
}

__device__ __forceinline__ int tile_pair_index(int ti, int tj, int T) {
  return ti * T - (ti * (ti - 1)) / 2 + (tj - ti);
}

template <typename ST>
__global__ void __launch_bounds__(256)
gram_tree(const ST* __restrict__ sums, int ntp, int n, int nblocks, ST* __restrict__ m_out) {
  const int T = (n + kTile - 1) / kTile;
  const long long nn = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nn;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e - (long long)i * n);  // row-major walk: coalesced reads
    if (i > j) continue;
    const int ti = i / kTile, tj = j / kTile;
    const int off = (i - ti * kTile) * kTile + (j - tj * kTile);
    const long long base = (long long)tile_pair_index(ti, tj, T) * (kTile * kTile) + off;
    const long long bstride = (long long)ntp * kTile * kTile;
    ST slot[16];
    for (int b = 0; b < nblocks; ++b) slot[b] = sums[b * bstride + base];
    for (int width = 1; width < nblocks; width *= 2)
      for (int b = 0; b + width < nblocks; b += 2 * width) slot[b] = st_add<ST>(slot[b], slot[b + width]);
    m_out[(long long)j * n + i] = slot[0];
    m_out[(long long)i * n + j] = slot[0];
  }
}

// Cross-rank combine for the multi-GPU path: the allgathered per-block sums
// of all ranks ([nblocks][n][n], global block order) go through the same tree.
__global__ void block_tree_f64(const double* __restrict__ blocks, int nblocks, int n,
                               double* __restrict__ m_out) {
  const long long nn = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nn;
       e += (long long)gridDim.x * blockDim.x) {
    double slot[16];
    for (int b = 0; b < nblocks; ++b) slot[b] = blocks[b * nn + e];
    for (int width = 1; width < nblocks; width *= 2)
      for (int b = 0; b + width < nblocks; b += 2 * width) slot[b] += slot[b + width];
    m_out[e] = slot[0];
  }
}

__global__ void block_tree_dd(const double2* __restrict__ blocks, int nblocks, int n,
                              double2* __restrict__ m_out) {
  const long long nn = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nn;
       e += (long long)gridDim.x * blockDim.x) {
    dd slot[16];
    for (int b = 0; b < nblocks; ++b) {
      const double2 v = blocks[b * nn + e];
      slot[b] = dd_make(v.x, v.y);
    }
    for (int width = 1; width < nblocks; width *= 2)
      for (int b = 0; b + width < nblocks; b += 2 * width) slot[b] = dd_add(slot[b], slot[b + width]);
    m_out[e] = make_double2(slot[0].hi, slot[0].lo);
  }
}

__global__ void mirror_upper(double* __restrict__ m, int n) {
  const long long nn = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nn;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / n), i = (int)(e % n);
    if (i > j) m[e] = m[(long long)i * n + j];
  }
}

// ---------------------------------------------------------------------------
// Host-side launchers (called by the engine, engine.cu).
cudaError_t launch_mirror_upper(double* m, int n, cudaStream_t st) {
  const long long nn = (long long)n * n;
  int grid = (int)((nn + 255) / 256);
  if (grid > 4 * 148) grid = 4 * 148;
  mirror_upper<<<grid, 256, 0, st>>>(m, n);
  return cudaGetLastError();
}

size_t gram_smem_bytes(bool dd) {
  return dd ? 2 * kKC * kLDC * sizeof(double) : 2 * 2 * kTile * kLDK * sizeof(double);
}

cudaError_t launch_gram_f32(const float* a, long long lda, int n, const int2* tiles, int ntp,
                            const longlong2* splits, int nsplit, double* partials,
                            cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gram_f32_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)gram_smem_bytes(false));
    configured = true;
  }
  dim3 grid(ntp, nsplit);
  gram_f32_dmma<<<grid, 128, gram_smem_bytes(false), st>>>(a, lda, n, tiles, splits, partials, ntp);
  return cudaGetLastError();
}

cudaError_t launch_gram_dd(const double* a, long long lda, int n, const int2* tiles, int ntp,
                           const longlong2* splits, int nsplit, double2* partials,
                           cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gram_f64_dd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)gram_smem_bytes(true));
    configured = true;
  }
  dim3 grid(ntp, nsplit);
  gram_f64_dd<<<grid, 256, gram_smem_bytes(true), st>>>(a, lda, n, tiles, splits, partials, ntp);
  return cudaGetLastError();
}

template <typename ST>
static cudaError_t combine_t(const ST* partials, int ntp, int n, const int* block_split_begin, int nblocks,
                             ST* sums, ST* m_out, cudaStream_t st) {
  dim3 g1(ntp, (kTile * kTile) / 256, nblocks);
  gram_block_sums<ST><<<g1, 256, 0, st>>>(partials, ntp, block_split_begin, sums);
  const long long nn = (long long)n * n;
  int grid = (int)((nn + 255) / 256);
  if (grid > 8 * 148) grid = 8 * 148;
  gram_tree<ST><<<grid, 256, 0, st>>>(sums, ntp, n, nblocks, m_out);
  return cudaGetLastError();
}

cudaError_t launch_gram_combine_f64(const double* partials, int ntp, int n, const int* block_split_begin,
                                    int nblocks, double* sums, double* m_out, cudaStream_t st) {
  return combine_t<double>(partials, ntp, n, block_split_begin, nblocks, sums, m_out, st);
}

cudaError_t launch_gram_combine_dd(const double2* partials, int ntp, int n, const int* block_split_begin,
                                   int nblocks, double2* sums, double2* m_out, cudaStream_t st) {
  return combine_t<double2>(partials, ntp, n, block_split_begin, nblocks, sums, m_out, st);
}

cudaError_t launch_block_tree(const void* blocks, int nblocks, int n, void* m_out, bool dd,
                              cudaStream_t st) {
  const long long nn = (long long)n * n;
  int grid = (int)((nn + 255) / 256);
  if (grid > 4 * 148) grid = 4 * 148;
  if (dd)
    block_tree_dd<<<grid, 256, 0, st>>>((const double2*)blocks, nblocks, n, (double2*)m_out);
  else
    block_tree_f64<<<grid, 256, 0, st>>>((const double*)blocks, nblocks, n, (double*)m_out);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace mpsvd
