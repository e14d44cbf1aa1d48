// K1 / K2: the higher-precision Gram product M = A^T A.
//
// Reference semantics: partitioned_gram (proj/src/parallel_gram.cpp:79-112)
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

// fp32 -> fp64 widening on the integer pipe. cvt.f64.f32 issues on the XU
// pipe, which the first K1 version saturated (98.7% XU, 61% DMMA in
// profiles/r01_gram_f32_v0.txt). For zero and normal numbers the widened
// value is a re-biased exponent and a shifted mantissa; subnormals, inf and
// NaN take the cvt path (warp-uniform vote per chunk).
__device__ __forceinline__ double widen_f32_alu(float x) {
  const uint32_t u = __float_as_uint(x), mag = u & 0x7fffffffu;
  const uint32_t hi = (mag ? (mag >> 3) + 0x38000000u : 0u) | (u & 0x80000000u);
  return __hiloint2double((int)hi, (int)(u << 29));
}
__device__ __forceinline__ bool f32_needs_cvt(float x) {  // subnormal, inf or NaN
  const uint32_t mag = __float_as_uint(x) & 0x7fffffffu;
  return (mag - 0x00800000u) >= 0x7f000000u && mag != 0u;
}

// Diagonal 64x64 tile: the 36 upper 8x8 blocks (i <= j over the 8 column
// groups) split 9 per warp, so the four warps (one per SM sub-partition)
// issue the same number of DMMAs. In a Gram tile the A fragment of group c
// (A[g][t] = X[k+t][8c+g]) equals its B fragment, so a warp loads each group
// it touches once per k-step.
//   W0: groups 0-3 minus (3,3)   W1: (3,3) + {0..3}x{4,5}
//   W2: (4,4) + {0..3}x{6,7}     W3: groups 4-7 minus (4,4)
__host__ __device__ constexpr int diag_pair(int w, int k, int e) {
  constexpr unsigned char t[4][9][2] = {
      {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}},
      {{3, 3}, {0, 4}, {1, 4}, {2, 4}, {3, 4}, {0, 5}, {1, 5}, {2, 5}, {3, 5}},
      {{4, 4}, {0, 6}, {1, 6}, {2, 6}, {3, 6}, {0, 7}, {1, 7}, {2, 7}, {3, 7}},
      {{5, 5}, {6, 6}, {7, 7}, {4, 5}, {4, 6}, {4, 7}, {5, 6}, {5, 7}, {6, 7}}};
  return t[w][k][e];
}

template <int W>
struct DiagSet {
  __host__ __device__ static constexpr int pi(int k) { return diag_pair(W, k, 0); }
  __host__ __device__ static constexpr int pj(int k) { return diag_pair(W, k, 1); }
  __host__ __device__ static constexpr bool uses(int c) {
    for (int k = 0; k < 9; ++k)
      if (pi(k) == c || pj(k) == c) return true;
    return false;
  }
};

// One K1 CTA body. MODE 0..3: warp MODE of a diagonal tile; MODE 4: any warp
// of an off-diagonal tile (2x2 warps, each 4x4 blocks of 8x8).
template <int MODE>
__device__ __forceinline__ void gram_f32_body(const float* __restrict__ a, long long lda, int n, int c0, int c1,
                                              long long r0, long long r1, double* __restrict__ out,
                                              double* __restrict__ smem) {
  constexpr bool kDiag = MODE < 4;
  constexpr int kNcol = kDiag ? kTile : 2 * kTile;
  constexpr int kNiter = kNcol / 4;  // 16 or 32 columns staged per warp
  constexpr int kNacc = kDiag ? 9 : 16;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wi = warp >> 1, wj = warp & 1;
  const int g = lane >> 2, t = lane & 3;

  double acc[kNacc][2];
#pragma unroll
  for (int k = 0; k < kNacc; ++k) acc[k][0] = acc[k][1] = 0.0;

  // Thread -> (column, row) of a chunk: warp w, iteration it loads column
  // 4*it+w, rows 0..31 -> one 128-byte segment per warp per iteration.
  float pre[kNiter];
  // columns of this tile present in A (CTA-uniform): n is normally a
  // multiple of 64, so only the last row chunk of a split needs row checks
  const bool cols_full = (kDiag ? c0 : c1) + kTile <= n;
  const float* abase = a + (long long)(c0 + warp) * lda + lane;
  const float* bbase = a + (long long)(c1 + warp) * lda + lane;
  auto load_chunk = [&](long long kr) {
    if (cols_full && kr + kKC <= r1) {
#pragma unroll
      for (int it = 0; it < kNiter; ++it) {
        const float* p = (it < 16 ? abase : bbase) + (long long)(4 * (it & 15)) * lda + kr;
        pre[it] = __ldg(p);
      }
    } else {
#pragma unroll
      for (int it = 0; it < kNiter; ++it) {
        const int lc = it * 4 + warp;
        const int gc = lc < kTile ? c0 + lc : c1 + (lc - kTile);
        const long long row = kr + lane;
        pre[it] = (gc < n && row < r1) ? __ldg(a + (long long)gc * lda + row) : 0.0f;
      }
    }
  };
  auto store_chunk = [&](double* buf) {
    bool special = false;
#pragma unroll
    for (int it = 0; it < kNiter; ++it) special |= f32_needs_cvt(pre[it]);
    if (__any_sync(0xffffffffu, special)) {
#pragma unroll
      for (int it = 0; it < kNiter; ++it) buf[(it * 4 + warp) * kLDK + lane] = (double)pre[it];
    } else {
#pragma unroll
      for (int it = 0; it < kNiter; ++it) buf[(it * 4 + warp) * kLDK + lane] = widen_f32_alu(pre[it]);
    }
  };

  const long long nchunks = (r1 - r0 + kKC - 1) / kKC;
  double* buf0 = smem;
  double* buf1 = smem + kNcol * kLDK;
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
#pragma unroll(kDiag ? 2 : 4)
    for (int kk = 0; kk < kKC; kk += 4) {
      if constexpr (kDiag) {
        double f[8];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (DiagSet<MODE>::uses(c)) f[c] = cur[(8 * c + g) * kLDK + kk + t];
#pragma unroll
        for (int k = 0; k < 9; ++k)
          dmma_8x8x4(acc[k][0], acc[k][1], f[DiagSet<MODE>::pi(k)], f[DiagSet<MODE>::pj(k)]);
      } else {
        double fa[4], fb[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) fa[mi] = cur[(32 * wi + 8 * mi + g) * kLDK + kk + t];
#pragma unroll
        for (int nj = 0; nj < 4; ++nj) fb[nj] = cur[(kTile + 32 * wj + 8 * nj + g) * kLDK + kk + t];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj) dmma_8x8x4(acc[mi * 4 + nj][0], acc[mi * 4 + nj][1], fa[mi], fb[nj]);
      }
    }
    if (more) store_chunk(nxt);
    __syncthreads();
  }

  // Epilogue: row-major 64x64 partial tile; entries below the diagonal of a
  // diagonal tile are never read by gram_combine.
#pragma unroll
  for (int k = 0; k < kNacc; ++k) {
    int r, c;
    if constexpr (kDiag) {
      r = 8 * DiagSet<MODE>::pi(k) + g;
      c = 8 * DiagSet<MODE>::pj(k) + 2 * t;
    } else {
      r = 32 * wi + 8 * (k >> 2) + g;
      c = 32 * wj + 8 * (k & 3) + 2 * t;
    }
    double2 v;
    v.x = acc[k][0];
    v.y = acc[k][1];
    *reinterpret_cast<double2*>(out + r * kTile + c) = v;
  }
}

// ---------------------------------------------------------------------------
// K1 launches: diagonal tiles (36 DMMA blocks per k-step, ~100 registers,
// 37 KB smem -> 4 CTAs per SM) and off-diagonal tiles (64 blocks, 254
// registers, 74 KB -> 2 CTAs per SM) are separate kernels so that each gets
// its own occupancy. blockIdx.x indexes `tp_list` (tile pair ids), blockIdx.y
// the row split; partial tiles land at (split * ntp + tp).
__global__ void __launch_bounds__(128, 4)
gram_f32_diag(const float* __restrict__ a, long long lda, int n, const int2* __restrict__ tiles,
              const int* __restrict__ tp_list, const longlong2* __restrict__ splits,
              double* __restrict__ partials, int ntp) {
  extern __shared__ __align__(16) double smem_k1[];
  const int tp = tp_list[blockIdx.x], s = blockIdx.y;
  const int c0 = tiles[tp].x * kTile;
  const long long r0 = splits[s].x, r1 = splits[s].y;
  double* out = partials + ((long long)s * ntp + tp) * (kTile * kTile);
  switch (threadIdx.x >> 5) {  // warp-uniform: warp w runs on sub-partition w
    case 0: gram_f32_body<0>(a, lda, n, c0, c0, r0, r1, out, smem_k1); break;
    case 1: gram_f32_body<1>(a, lda, n, c0, c0, r0, r1, out, smem_k1); break;
    case 2: gram_f32_body<2>(a, lda, n, c0, c0, r0, r1, out, smem_k1); break;
    default: gram_f32_body<3>(a, lda, n, c0, c0, r0, r1, out, smem_k1); break;
  }
}

__global__ void __launch_bounds__(128, 2)
gram_f32_offdiag(const float* __restrict__ a, long long lda, int n, const int2* __restrict__ tiles,
                 const int* __restrict__ tp_list, const longlong2* __restrict__ splits,
                 double* __restrict__ partials, int ntp) {
  extern __shared__ __align__(16) double smem_k1[];
  const int tp = tp_list[blockIdx.x], s = blockIdx.y;
  const int2 tij = tiles[tp];
  const long long r0 = splits[s].x, r1 = splits[s].y;
  double* out = partials + ((long long)s * ntp + tp) * (kTile * kTile);
  gram_f32_body<4>(a, lda, n, tij.x * kTile, tij.y * kTile, r0, r1, out, smem_k1);
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

cudaError_t launch_gram_f32(const float* a, long long lda, int n, const int2* tiles, int ntp, const int* tp_diag,
                            int ndiag, const int* tp_off, int noff, const longlong2* splits, int nsplit,
                            double* partials, cudaStream_t st) {
  const size_t smem_d = 2 * kTile * kLDK * sizeof(double), smem_o = 2 * smem_d;
  // the opt-in is a per-device (per-context) attribute: set it on every launch
  cudaFuncSetAttribute(gram_f32_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
  cudaFuncSetAttribute(gram_f32_offdiag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_o);
  if (ndiag > 0)
    gram_f32_diag<<<dim3(ndiag, nsplit), 128, smem_d, st>>>(a, lda, n, tiles, tp_diag, splits, partials, ntp);
  if (noff > 0)
    gram_f32_offdiag<<<dim3(noff, nsplit), 128, smem_o, st>>>(a, lda, n, tiles, tp_off, splits, partials, ntp);
  return cudaGetLastError();
}

cudaError_t launch_gram_dd(const double* a, long long lda, int n, const int2* tiles, int ntp,
                           const longlong2* splits, int nsplit, double2* partials,
                           cudaStream_t st) {
  cudaFuncSetAttribute(gram_f64_dd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem_bytes(true));
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
