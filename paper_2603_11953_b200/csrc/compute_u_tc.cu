// K7 on the 5th-generation tensor cores: U = A * W for fp32 A (m x n,
// column-major) and n <= 128, W = V Sigma^-1 (thinsvd.cpp:110-113).
//
// fp32 operands are split into three bf16 pieces, x = x0 + x1 + x2 (each
// piece the bf16 rounding of the remainder; 3 x 8 significand bits cover
// fp32's 24), and U accumulates the six piece products whose weight is at
// least 2^-16 of the leading one,
//     A2W0 + A1W1 + A0W2 + A1W0 + A0W1 + A0W0,
// in one fp32 TMEM accumulator. Every bf16 x bf16 product is exact; the
// dropped terms (A1W2, A2W1, A2W2) are <= 2^-24 relative, the size of the
// fp32 rounding the reference's own U accumulation commits per term
// (dense.cpp:83-96), so U keeps working-precision accuracy.
//
// Structure (one persistent CTA per SM, 19 warps, warp-specialised):
//   warps 16-17 load  : stream fp32 A chunks (128 rows x 16 columns) with
//                       16-byte cp.async, whole 128-byte lines per 8 lanes,
//                       kDepth chunks ahead; completion is signalled with
//                       cp.async.mbarrier.arrive (no thread waits on loads)
//   warps 0-7 convert : staging fp32 -> three bf16 planes in the UMMA
//                       MN-major no-swizzle layout (8x8 core matrices), one
//                       generic->async proxy fence per chunk. The loads are
//                       kept out of these warps: fence.proxy.async waits for
//                       the issuing thread's outstanding cp.async, which
//                       serialised converter warps that also loaded on the
//                       full memory latency (profiles/r01_av_tc_notes.md).
//   warp 18 MMA       : W pieces once (one bulk copy); one thread issues 6
//                       tcgen05.mma (M=128, N=np, K=16)
//                       per chunk into a double-buffered TMEM accumulator
//   warps 8-15 epilogue: tcgen05.ld 32x32b -> coalesced column stores of U
//                       (two warps per TMEM lane quarter, alternate 16-column
//                       groups; branch-free strided stores for full groups)
// The encodings (descriptors, instruction descriptor, TMEM load shape) are
// the ones checked by tools/microbench/umma_test.cu on the B200.
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

#ifndef TM_LOAD_WARPS
#define TM_LOAD_WARPS 2  // loader warps of the TMEM variant (4 measured 5% slower)
#endif

namespace mpsvd {
namespace dev {
namespace tc {

constexpr int kBM = 128;                          // rows per tile = UMMA M
constexpr int kKC = 16;                           // K per chunk = UMMA K
constexpr int kMaxDepth = 8;                      // fp32 A chunks in flight per CTA (staging ring)
constexpr int kStageBytes = kBM * kKC * 4;        // fp32 chunk: 8 KB
constexpr int kPlaneBytes = kBM * kKC * 2;        // one bf16 piece of a chunk: 4096
constexpr int kConvWarps = 8, kEpiWarps = 8;      // converters: warps 0-7; epilogue: warps 8-15
constexpr int kLoadWarps = 2;                     // A loaders: warps 16-17
constexpr int kWarpLoad0 = 16, kWarpMma = 18;
constexpr int kThreads = 608;
constexpr int kPlanes = 8;                        // max bf16 chunk slots = one per active converter warp
constexpr int kSmemLimit = 227 * 1024;

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // sm100 descriptor version; base offset 0, no swizzle
  return d;
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(saddr(bar))
               : "memory");
}

// x = h + m + l, each a bf16 (rounded remainders); packs 2 values per word.
__device__ __forceinline__ void split3(float x0, float x1, uint32_t& h, uint32_t& m, uint32_t& l) {
  const __nv_bfloat162 bh = __floats2bfloat162_rn(x0, x1);
  const float2 fh = __bfloat1622float2(bh);
  const float r0 = x0 - fh.x, r1 = x1 - fh.y;
  const __nv_bfloat162 bm = __floats2bfloat162_rn(r0, r1);
  const float2 fm = __bfloat1622float2(bm);
  const __nv_bfloat162 bl = __floats2bfloat162_rn(r0 - fm.x, r1 - fm.y);
  h = *reinterpret_cast<const uint32_t*>(&bh);
  m = *reinterpret_cast<const uint32_t*>(&bm);
  l = *reinterpret_cast<const uint32_t*>(&bl);
}

// Byte offset of (mn, k) in an MN-major no-swizzle operand image whose MN
// extent is `mn_ext`: 8x8 core matrices of 128 B (mn contiguous, 16 B per k
// row), MN groups adjacent (SBO = 128 B), K groups `mn_ext/8 * 128` apart (LBO).
__host__ __device__ __forceinline__ uint32_t mn_major_off(int mn, int k, int mn_ext) {
  return (uint32_t)((((k >> 3) * (mn_ext >> 3) + (mn >> 3)) << 7) + ((k & 7) << 4) + ((mn & 7) << 1));
}

}  // namespace tc

// W (n x n, fp32, row-major rows of ldw = W^T buffer of finish_columns) ->
// three bf16 planes, each the np x np (K x N, N-major) smem image.
__global__ void av_tc_prep_w(const float* __restrict__ w, int ldw, int n, int np, __nv_bfloat16* __restrict__ planes,
                             const DevStatus* __restrict__ status) {
  if (status && status->status != kOk) return;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= np * np) return;
  const int k = idx / np, c = idx - k * np;
  const float x = (k < n && c < n) ? w[(long long)k * ldw + c] : 0.0f;
  uint32_t h, m, l;
  tc::split3(x, 0.0f, h, m, l);
  const uint32_t off = tc::mn_major_off(c, k, np) >> 1;  // in bf16 elements
  const size_t plane = (size_t)np * np;
  planes[off] = __ushort_as_bfloat16((unsigned short)(h & 0xFFFF));
  planes[plane + off] = __ushort_as_bfloat16((unsigned short)(m & 0xFFFF));
  planes[2 * plane + off] = __ushort_as_bfloat16((unsigned short)(l & 0xFFFF));
}

// dbg bit 2: CTA 0 accumulates per-phase cycle counts (converter warp 0,
// MMA thread, epilogue warp 8) into g_av_prof
__device__ unsigned long long g_av_prof[16];
#define AVP_T0() _t0 = (prof ? clock64() : 0ull)
#define AVP_ADD(i) do { if (prof) pacc[i] += clock64() - _t0; } while (0)

__global__ void __launch_bounds__(tc::kThreads, 1)
av_tc_f32(const float* __restrict__ a, long long lda, long long m, int n, int np,
          const __nv_bfloat16* __restrict__ wplanes, float* __restrict__ u, long long ldu,
          const DevStatus* __restrict__ status, int depth, int dbg) {
  // `depth` = staging slots = bf16 plane slots = active converter warps (4 or
  // 8): every slot belongs to one converter warp, so each mbarrier is waited
  // on by a single consumer that is never more than one phase behind.
  using namespace tc;
  if (status && status->status != kOk) return;
  extern __shared__ __align__(1024) unsigned char smem_tc[];
  const int nkc = np / kKC;
  const uint32_t wbytes = 3u * np * np * 2u;
  unsigned char* wsm = smem_tc;
  unsigned char* psm = wsm + ((wbytes + 1023) & ~1023u);
  unsigned char* ssm = psm + depth * 3 * kPlaneBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ssm + depth * kStageBytes);
  uint64_t* stage_full = bars;
  uint64_t* stage_empty = stage_full + depth;
  uint64_t* plane_full = stage_empty + depth;
  uint64_t* plane_empty = plane_full + depth;
  uint64_t* acc_full = plane_empty + depth;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* w_full = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long ntiles = (m + kBM - 1) / kBM;
  const bool prof = (dbg & 4) && blockIdx.x == 0 && (lane == 0) && (warp == 0 || warp == kWarpMma || warp == 8);
  const int my_tiles = (int)(ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  const int nchunks = my_tiles * nkc;
  const unsigned long long t_start = prof ? clock64() : 0ull;
  unsigned long long _t0 = 0, pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const uint32_t tcols = np * 2 <= 32 ? 32 : np * 2 <= 64 ? 64 : np * 2 <= 128 ? 128 : 256;

  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) {
      mbar_init(&stage_full[i], kLoadWarps * 32);  // one cp.async-completion arrive per loader thread
      mbar_init(&stage_empty[i], 1);               // the converter warp of the chunk
    }
    for (int i = 0; i < depth; ++i) {
      mbar_init(&plane_full[i], 1);
      mbar_init(&plane_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kEpiWarps);
    }
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == kWarpMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(saddr(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp >= kWarpLoad0 && warp < kWarpLoad0 + kLoadWarps) {
    // loader thread lt fetches 16-byte pieces q = lt + 64 i (i < 8) of each
    // chunk: column q / 32, rows 4 (q % 32) .. +3 (8 lanes read a whole
    // 128-byte line); the piece is written where its converter lane reads
    // it: [item][half][lane] x 16 B.
    const int lt = threadIdx.x - kWarpLoad0 * 32;
    int dst_off[8], col_off[8], row_off[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int q = lt + 64 * i, c = q >> 5, p = q & 31;
      const int rg = p >> 1, half = p & 1, kg = c >> 3, kl = c & 7;
      const int item = (rg >> 2) + 4 * kg, clane = (rg & 3) * 8 + kl;
      dst_off[i] = ((item * 2 + half) * 32 + clane) * 16;
      col_off[i] = c;
      row_off[i] = p * 4;
    }
    long long row0 = (long long)blockIdx.x * kBM;
    const long long row_step = (long long)gridDim.x * kBM;
    int kc = 0, slot = 0;
    unsigned ph = 0;
    for (int g = 0; g < nchunks; ++g) {
      mbar_wait(&stage_empty[slot], ph ^ 1);
      unsigned char* dst = ssm + slot * kStageBytes;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int col = kc * kKC + col_off[i];
        const long long row = row0 + row_off[i];
        const bool ok = col < n && row < m;  // m % 4 == 0: a 16-byte piece is all in or all out
        cp_async16_zfill(dst + dst_off[i], ok ? a + (long long)col * lda + row : a, ok);
      }
      cp_async_mbar_arrive(&stage_full[slot]);
      if (++kc == nkc) {
        kc = 0;
        row0 += row_step;
      }
      if (++slot == depth) {
        slot = 0;
        ph ^= 1;
      }
    }
    cp_async_wait<0>();
  } else if (warp == kWarpMma) {
    if (lane == 0) {
      // D f32, A/B bf16, both MN-major, N = np, M = 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                             ((uint32_t)(np >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
      const uint32_t a_lbo = (kBM / 8) * 128, w_lbo = (uint32_t)(np / 8) * 128;
      const uint32_t wbase = saddr(wsm), pbase = saddr(psm);
      const uint32_t wplane = (uint32_t)np * np * 2u;
      // (A piece, W piece), smallest products first
      const int pa[6] = {2, 1, 0, 1, 0, 0}, pw[6] = {0, 1, 2, 0, 1, 0};
      mbar_expect_tx(w_full, wbytes);
      bulk_g2s(wsm, wplanes, wbytes, w_full);
      mbar_wait(w_full, 0);
      int ps = 0, ab = 0;
      unsigned pph = 0, aph = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        { AVP_T0(); mbar_wait(&acc_empty[ab], aph ^ 1); AVP_ADD(0); }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t d = tmem + (uint32_t)ab * (tcols / 2);
        for (int kc = 0; kc < nkc; ++kc) {
          { AVP_T0(); mbar_wait(&plane_full[ps], pph); AVP_ADD(1); }
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            const uint64_t ad = umma_desc(pbase + (uint32_t)(ps * 3 + pa[q]) * kPlaneBytes, a_lbo, 128);
            const uint64_t bd = umma_desc(wbase + (uint32_t)pw[q] * wplane + (uint32_t)kc * 2u * w_lbo, w_lbo, 128);
            if (!(dbg & 2)) umma_bf16(d, ad, bd, idesc, (kc > 0 || q > 0) ? 1u : 0u);
          }
          umma_commit(&plane_empty[ps]);
          if (++ps == depth) {
            ps = 0;
            pph ^= 1;
          }
        }
        umma_commit(&acc_full[ab]);
        if (++ab == 2) {
          ab = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp < kConvWarps) {
    // Warp-per-chunk: converter warp w (< depth) converts chunks w, w + depth,
    // ... from staging slot w into its own plane slot w, so the warps'
    // barrier and proxy-fence latencies overlap instead of adding up per
    // chunk. Lane (rgl, kl) handles items i = 0..7: 8 rows (row group
    // rgl + 4 (i & 3)) of column 8 (i >> 2) + kl; reads are [item][half][lane]
    // x 16 B and each 8-lane phase writes one contiguous 128-byte core-matrix
    // row: conflict-free.
    if (warp < depth) {
      const int kl = lane & 7, rgl = lane >> 3;
      unsigned char* dst = psm + warp * 3 * kPlaneBytes;
      const unsigned char* src = ssm + warp * kStageBytes + lane * 16;
      unsigned ph = 0;
      for (int g = warp; g < nchunks; g += depth) {
        { AVP_T0(); mbar_wait(&stage_full[warp], ph); mbar_wait(&plane_empty[warp], ph ^ 1); AVP_ADD(2); }
        AVP_T0();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float4 x[4], y[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int i = hh * 4 + j;
            x[j] = *reinterpret_cast<const float4*>(src + (i * 2 + 0) * 512);
            y[j] = *reinterpret_cast<const float4*>(src + (i * 2 + 1) * 512);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int i = hh * 4 + j;
            uint4 h, mm, l;
            split3(x[j].x, x[j].y, h.x, mm.x, l.x);
            split3(x[j].z, x[j].w, h.y, mm.y, l.y);
            split3(y[j].x, y[j].y, h.z, mm.z, l.z);
            split3(y[j].z, y[j].w, h.w, mm.w, l.w);
            const uint32_t off = mn_major_off((rgl + 4 * (i & 3)) * 8, (i >> 2) * 8 + kl, kBM);
            *reinterpret_cast<uint4*>(dst + off) = h;
            *reinterpret_cast<uint4*>(dst + kPlaneBytes + off) = mm;
            *reinterpret_cast<uint4*>(dst + 2 * kPlaneBytes + off) = l;
          }
        }
        AVP_ADD(3);
        AVP_T0();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&stage_empty[warp]);
          mbar_arrive(&plane_full[warp]);
        }
        ph ^= 1;
        AVP_ADD(5);
      }
    }
  } else if (warp < kConvWarps + kEpiWarps) {
    // epilogue: TMEM lane quarter = warp % 4; e selects alternate 16-column groups
    const int q = warp & 3, e = (warp - kConvWarps) >> 2;
    int ab = 0;
    unsigned aph = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      { AVP_T0(); mbar_wait(&acc_full[ab], aph); AVP_ADD(6); }
      AVP_T0();
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const long long row = tile * kBM + q * 32 + lane;
      const bool row_ok = row < m && !(dbg & 1);
      float* base = u + row;
      for (int c0 = 16 * e; c0 < np; c0 += 32) {
        uint32_t r[16];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)ab * (tcols / 2) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
            "[%16];\n"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (row_ok) {
          float* p = base + (long long)c0 * ldu;
          if (c0 + 16 <= n) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              *p = __uint_as_float(r[j]);
              p += ldu;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c0 + j < n) p[(long long)j * ldu] = __uint_as_float(r[j]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
      AVP_ADD(7);
      if (++ab == 2) {
        ab = 0;
        aph ^= 1;
      }
    }
  }
  if (prof) {
    g_av_prof[8 + (warp == 0 ? 0 : warp == 8 ? 1 : 2)] = clock64() - t_start;
    for (int i = 0; i < 8; ++i)
      if (pacc[i]) g_av_prof[i] = pacc[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == kWarpMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tcols));
}


// ---------------------------------------------------------------------------
__device__ __forceinline__ void nbar_sync_k7(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// K7, TMEM variant: the bf16 pieces of A are written to tensor memory with
// tcgen05.st (thread = row) and fed to the MMA as its A operand (K-major in
// TMEM, two K-neighbours per 32-bit column, low half = even k; encoding
// checked by tools/microbench/umma_tmem_a.cu). No shared-memory planes and
// no generic->async proxy fence; the freed shared memory deepens the fp32
// staging ring. Roles:
//   warps 0-15  converters, four groups of four (one warp per TMEM lane
//               quarter); group g converts chunks g, g + 4, ... into TMEM
//               A slots {g, g + 4} (each slot has one owner group)
//   warps 16-23 epilogue (as in av_tc_f32)
//   warps 24-25 loaders: fp32 chunk [16 columns][128 rows] by cp.async
//   warp 26     W pieces (bulk copy) + MMA issue
namespace tm {
#ifndef TM_GROUPS
#define TM_GROUPS 4  // converter groups (4 warps each); 2 left the MMA waiting for A slots (C4 ncu)
#endif
constexpr int kGroups = TM_GROUPS;
constexpr int kASlots = 2 * kGroups;  // TMEM A slots (24 columns each: 3 pieces x 8)
constexpr int kACols = 3 * 8;
constexpr int kConvW = 4 * kGroups, kEpi0 = kConvW;  // converters: warps 0 .. kConvW-1, then 8 epilogue warps
constexpr int kLoad0 = kEpi0 + 8, kLoadWarps = TM_LOAD_WARPS, kMma = kLoad0 + kLoadWarps;
constexpr int kThreads = 32 * (kMma + 1);
constexpr int kPieces = 512 / (32 * kLoadWarps);  // 16-byte pieces per loader thread per chunk
}  // namespace tm

__global__ void __launch_bounds__(tm::kThreads, 1)
av_tc_tmem_f32(const float* __restrict__ a, long long lda, long long m, int n, int np,
               const __nv_bfloat16* __restrict__ wplanes, float* __restrict__ u, long long ldu,
               const DevStatus* __restrict__ status, int nstage, int acc_stride, int a_col0, int tcols) {
  using namespace tc;
  using namespace tm;
  if (status && status->status != kOk) return;
  extern __shared__ __align__(1024) unsigned char smem_tc[];
  const int nkc = np / kKC;
  const uint32_t wbytes = 3u * np * np * 2u;
  unsigned char* wsm = smem_tc;
  unsigned char* ssm = wsm + ((wbytes + 1023) & ~1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ssm + nstage * kStageBytes);
  uint64_t* stage_full = bars;
  uint64_t* stage_empty = stage_full + nstage;
  uint64_t* a_full = stage_empty + nstage;
  uint64_t* a_empty = a_full + kASlots;
  uint64_t* acc_full = a_empty + kASlots;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* w_full = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long ntiles = (m + kBM - 1) / kBM;
  const int my_tiles = (int)(ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  const int nchunks = my_tiles * nkc;
  const int kdbg = tcols >> 16;  // experiment switches (MPSVD_AV_DBG bits 4-6): 1 no MMA, 2 no U stores, 4 no split
  tcols &= 0xFFFF;
  const uint32_t zmask = (uint32_t)kdbg >> 8;  // 0 (kdbg < 256), unknown to the compiler

  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) {
      mbar_init(&stage_full[i], tm::kLoadWarps * 32);
      mbar_init(&stage_empty[i], 4);  // the four warps of the converting group
    }
    for (int i = 0; i < kASlots; ++i) {
      mbar_init(&a_full[i], 4);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kEpiWarps);
    }
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == tm::kMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(saddr(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp >= tm::kLoad0 && warp < tm::kLoad0 + tm::kLoadWarps) {
    // chunk = 16 columns x 128 rows fp32, column-major in the slot (512 B per
    // column): loader thread lt fetches pieces q = lt + 64 i, each 16 bytes of
    // one column, a warp a whole 512-byte column segment per instruction
    const int lt = threadIdx.x - tm::kLoad0 * 32;
    long long row0 = (long long)blockIdx.x * kBM;
    const long long row_step = (long long)gridDim.x * kBM;
    int kc = 0, slot = 0;
    unsigned ph = 0;
    for (int g = 0; g < nchunks; ++g) {
      mbar_wait(&stage_empty[slot], ph ^ 1);
      unsigned char* dst = ssm + slot * kStageBytes;
#pragma unroll
      for (int i = 0; i < tm::kPieces; ++i) {
        const int q = lt + 32 * tm::kLoadWarps * i, c = q >> 5, p = q & 31;
        const int col = kc * kKC + c;
        const long long row = row0 + p * 4;
        const bool ok = col < n && row < m;  // m % 4 == 0: a 16-byte piece is all in or all out
        cp_async16_zfill(dst + q * 16, ok ? a + (long long)col * lda + row : a, ok);
      }
      cp_async_mbar_arrive(&stage_full[slot]);
      if (++kc == nkc) {
        kc = 0;
        row0 += row_step;
      }
      if (++slot == nstage) {
        slot = 0;
        ph ^= 1;
      }
    }
    cp_async_wait<0>();
  } else if (warp == tm::kMma) {
    if (lane == 0) {
      // D f32, A bf16 K-major (TMEM), B bf16 MN-major (smem), N = np, M = 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(np >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      const uint32_t w_lbo = (uint32_t)(np / 8) * 128;
      const uint32_t wbase = saddr(wsm);
      const uint32_t wplane = (uint32_t)np * np * 2u;
      const int pa[6] = {2, 1, 0, 1, 0, 0}, pw[6] = {0, 1, 2, 0, 1, 0};
      mbar_expect_tx(w_full, wbytes);
      bulk_g2s(wsm, wplanes, wbytes, w_full);
      mbar_wait(w_full, 0);
      int ab = 0;
      unsigned aph = 0;
      int g = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        mbar_wait(&acc_empty[ab], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(ab * acc_stride);
        for (int kc = 0; kc < nkc; ++kc, ++g) {
          const int sl = g % kASlots;
          mbar_wait(&a_full[sl], (unsigned)((g / kASlots) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t at = tmem + (uint32_t)(a_col0 + sl * kACols);
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            if (kdbg & 1) break;
            const uint64_t bd = umma_desc(wbase + (uint32_t)pw[q] * wplane + (uint32_t)kc * 2u * w_lbo, w_lbo, 128);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                "r"(at + (uint32_t)(pa[q] * 8)), "l"(bd), "r"(idesc), "r"((kc > 0 || q > 0) ? 1u : 0u));
          }
          umma_commit(&a_empty[sl]);
        }
        umma_commit(&acc_full[ab]);
        if (++ab == 2) {
          ab = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp < tm::kConvW) {
    // converter group grp = warp / 4; quarter q = warp % 4 owns TMEM lanes
    // 32q .. 32q + 31 (rows of the tile)
    const int grp = warp >> 2, q = warp & 3;
    const int row = q * 32 + lane;
    int slot = grp % nstage;
    unsigned sph = (unsigned)((grp / nstage) & 1);
    // one warp of the group polls each mbarrier, the other three wait on the
    // group's named barrier (all 16 converter warps polling took ~40% of the
    // SM's issue slots, ncu c4)
    for (int g = grp; g < nchunks; g += kGroups) {
      const int sl = g % kASlots;
      if (q == 0) mbar_wait(&stage_full[slot], sph);
      nbar_sync_k7(1 + grp, 128);
      const float* src = reinterpret_cast<const float*>(ssm + slot * kStageBytes);
      float v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = src[c * kBM + row];  // consecutive lanes: consecutive rows
      uint32_t hp[8], mp[8], lp[8];
      if (kdbg & 4) {
#pragma unroll
        for (int c = 0; c < 8; ++c) hp[c] = mp[c] = lp[c] = __float_as_uint(v[2 * c]) ^ __float_as_uint(v[2 * c + 1]);
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) split3(v[2 * c], v[2 * c + 1], hp[c], mp[c], lp[c]);
      }
      // release the staging slot only once every lane's loads have returned:
      // an arrive right after the loads (lane 0, after __syncwarp) can
      // overtake loads still in flight, and the loaders then overwrite the
      // slot under them (measured on K1z's identical ring, gram_ozaki32.cu
      // release_a). The arrive count depends on a warp OR-reduction of a
      // runtime zero derived from all 16 values (via the last pieces).
      {
        const uint32_t dep = (lp[0] | lp[1] | lp[2] | lp[3]) | (lp[4] | lp[5] | lp[6] | lp[7]);
        const uint32_t z = __reduce_or_sync(0xffffffffu, dep & zmask);
        if (lane == 0)
          asm volatile(
              "{\n.reg .b32 cnt;\nadd.u32 cnt, %1, 1;\n"
              "mbarrier.arrive.shared::cta.b64 _, [%0], cnt;\n}\n" ::"r"(saddr(&stage_empty[slot])),
              "r"(z)
              : "memory");
      }
      slot += kGroups;
      if (slot >= nstage) {
        slot -= nstage;
        sph ^= 1;
      }
      if (q == 0) mbar_wait(&a_empty[sl], (unsigned)(((g / kASlots) & 1) ^ 1));
      nbar_sync_k7(1 + grp, 128);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a_col0 + sl * kACols);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta), "r"(hp[0]),
                   "r"(hp[1]), "r"(hp[2]), "r"(hp[3]), "r"(hp[4]), "r"(hp[5]), "r"(hp[6]), "r"(hp[7]));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta + 8u),
                   "r"(mp[0]), "r"(mp[1]), "r"(mp[2]), "r"(mp[3]), "r"(mp[4]), "r"(mp[5]), "r"(mp[6]), "r"(mp[7]));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta + 16u),
                   "r"(lp[0]), "r"(lp[1]), "r"(lp[2]), "r"(lp[3]), "r"(lp[4]), "r"(lp[5]), "r"(lp[6]), "r"(lp[7]));
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[sl]);
    }
  } else if (warp < tm::kEpi0 + kEpiWarps) {
    const int q = warp & 3, e = (warp - tm::kEpi0) >> 2;
    int ab = 0;
    unsigned aph = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      if (warp == tm::kEpi0) mbar_wait(&acc_full[ab], aph);  // one poller, the epilogue waits on barrier 5
      nbar_sync_k7(1 + kGroups, 32 * kEpiWarps);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const long long row = tile * kBM + q * 32 + lane;
      const bool row_ok = row < m;
      float* base = u + row;
      for (int c0 = 16 * e; c0 < np; c0 += 32) {
        uint32_t r[16];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * acc_stride + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
            "[%16];\n"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (row_ok && !(kdbg & 2)) {
          float* p = base + (long long)c0 * ldu;
          if (c0 + 16 <= n) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              *p = __uint_as_float(r[j]);
              p += ldu;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c0 + j < n) p[(long long)j * ldu] = __uint_as_float(r[j]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
      if (++ab == 2) {
        ab = 0;
        aph ^= 1;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == tm::kMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tcols));
}

// ---------------------------------------------------------------------------
bool av_tc_supported(const float* a, long long lda, long long m, int n, long long ldu) {
  (void)ldu;
  if (n < 1 || n > 128 || m < 1) return false;
  if (m % 4 != 0 || lda % 4 != 0) return false;  // 16-byte bulk copies of every column segment
  if (reinterpret_cast<uintptr_t>(a) % 16 != 0) return false;
  return true;
}

size_t av_tc_wplanes_bytes(int n) {
  const int np = (n + 15) / 16 * 16;
  return 3ull * np * np * 2ull;
}

// experiment switches of the shared-memory-plane variant (MPSVD_AV_PLANES=1,
// or any MPSVD_AV_DBG bit selects it) — MPSVD_AV_DBG: bit 0 skips the U stores, bit 1 the
// MMAs, bit 2 prints per-role cycle counts of CTA 0 (tools/av_probe.sh).
// Findings (C2, n = 64): loads + conversion alone take 0.089 ms of the
// 0.128 ms, and with loads, conversion, MMAs and stores all skipped the
// barrier hand-offs alone still take ~0.065 ms: the ring of mbarrier
// hand-offs (loader -> converter -> MMA -> epilogue, 8 slots deep, limited by
// shared memory) bounds K7 at small n, not HBM. An XOR-swizzled staging
// layout (conflict-free cp.async writes), 4 loader warps, packing the six
// products into four MMAs (N = 2n) and test_wait spinning were all measured
// slower or equal and not kept.
static int g_av_dbg = [] {
  const char* e = getenv("MPSVD_AV_DBG");
  return e ? atoi(e) : 0;
}();

cudaError_t launch_av_tc_f32(const float* a, long long lda, long long m, int n, const float* w, void* wplanes,
                             float* u, long long ldu, const DevStatus* status, int sm_count, cudaStream_t st,
                             bool prep) {
  using namespace tc;
  const int np = (n + 15) / 16 * 16;
  const int ldw = av_ldw(n);
  const int prep_threads = 256;
  if (prep)
    av_tc_prep_w<<<(np * np + prep_threads - 1) / prep_threads, prep_threads, 0, st>>>(
        w, ldw, n, np, reinterpret_cast<__nv_bfloat16*>(wplanes), status);
  const size_t wbytes = ((size_t)3 * np * np * 2 + 1023) & ~(size_t)1023;
  static const bool planes = getenv("MPSVD_AV_PLANES") != nullptr;  // the shared-memory-plane variant
  if (!planes && !(g_av_dbg & 7)) {
    // TMEM variant: accumulators [0, 2 acc_stride), A slots after them
    const int acc_stride = np <= 32 ? 32 : np <= 64 ? 64 : 128;
    const int a_col0 = 2 * acc_stride;
    const int need = a_col0 + tm::kASlots * tm::kACols;
    const int tcols = need <= 128 ? 128 : need <= 256 ? 256 : 512;
    int nstage = (int)((kSmemLimit - wbytes - 1024) / kStageBytes);
    static const int stage_cap = getenv("MPSVD_AV_STAGES") ? atoi(getenv("MPSVD_AV_STAGES")) : 16;
    if (nstage > stage_cap) nstage = stage_cap;
    if (nstage < tm::kGroups) return cudaErrorInvalidConfiguration;
    const size_t smem = wbytes + (size_t)nstage * kStageBytes + 1024;
    cudaError_t e = cudaFuncSetAttribute(av_tc_tmem_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long ntiles = (m + kBM - 1) / kBM;
    const int grid = (int)(ntiles < sm_count ? ntiles : sm_count);
    av_tc_tmem_f32<<<grid, tm::kThreads, smem, st>>>(a, lda, m, n, np, reinterpret_cast<const __nv_bfloat16*>(wplanes),
                                                 u, ldu, status, nstage, acc_stride, a_col0,
                                                 tcols | (((g_av_dbg >> 4) & 7) << 16));
    return cudaGetLastError();
  }
  // one staging slot + one plane slot per active converter warp
  int depth = kConvWarps;
  auto smem_for = [&](int d) { return wbytes + (size_t)d * (3 * kPlaneBytes + kStageBytes) + 512; };
  while (depth > 1 && smem_for(depth) > (size_t)kSmemLimit) depth /= 2;
  const size_t smem = smem_for(depth);
  if (smem > (size_t)kSmemLimit || depth < 2) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(av_tc_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long ntiles = (m + kBM - 1) / kBM;
  const int grid = (int)(ntiles < sm_count ? ntiles : sm_count);
  if (g_av_dbg & 4) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbolAsync(g_av_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
  }
  av_tc_f32<<<grid, kThreads, smem, st>>>(a, lda, m, n, np, reinterpret_cast<const __nv_bfloat16*>(wplanes), u, ldu,
                                          status, depth, g_av_dbg);
  if (g_av_dbg & 4) {
    unsigned long long h[16];
    cudaMemcpyFromSymbolAsync(h, g_av_prof, sizeof(h), 0, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr,
            "av_tc prof (cycles, CTA 0): mma: acc_empty %llu plane_full %llu | conv: data %llu split+issue %llu "
            "plane_empty %llu store+fence %llu | epi: acc_full %llu ld+store %llu | total conv %llu epi %llu mma %llu\n",
            h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9], h[10]);
  }
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace mpsvd
