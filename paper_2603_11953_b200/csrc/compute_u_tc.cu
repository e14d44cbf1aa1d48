// K7 on the 5th-generation tensor cores: U = A * W for fp32 A (m x n,
// column-major) and n <= 128, W = V Sigma^-1 (thinsvd.cpp:110-113).
//
// A is split into two fp16 pieces and W into three, after an exact
// power-of-two scaling: column c of A by 2^-s_c and row c of W by 2^s_c (2^s_c >= the
// column norm sqrt(M_cc) / 2^14, so every scaled entry of A is < 2^14), and
// column j of W by 2^-t_j (its largest scaled entry < 2^14) with U's column
// j multiplied back by 2^t_j in the epilogue. a = a0 + a1 (a0 = fp16(a),
// a1 = fp16(a - a0)) carries 22 significand bits, w = w0 + w1 + w2 all of
// binary32's 24; U accumulates the four piece products A1 W0 + A0 W2 +
// A0 W1 + A0 W0 in one fp32 TMEM accumulator. Every fp16 x fp16 product is
// exact; the dropped A1 W1 and A1 W2 and A's representation error are
// ~2^-22 relative per term, below the error of the reference's own fp32
// accumulation (dense.cpp:83-96: up to n u with u = 2^-24), so U keeps
// working-precision accuracy (tests bound it by 2 n u |A||W| elementwise),
// and W is carried exactly, so an A whose entries fit 22 bits gives U =
// fl(A W) like the reference (the stacked-diagonal known answer,
// test_thinsvd.cpp: U = [I; 0] exactly). Entries below 2^-14 of the scaled
// range become fp16 subnormals: their absolute error stays below
// 2^-24 2^s_c, far under the bound. (The first version used three bf16
// pieces of both operands and six products: 14.6 ms at c4 against 12.7 ms
// with two fp16 pieces of each - which loses W's exactness.)
//
// Structure (one persistent CTA per SM, warp-specialised):
//   warps 0-15  converters, four groups of four (one warp per TMEM lane
//               quarter); group g converts chunks g, g + 4, ... (128 rows x
//               16 columns: thread = row) into TMEM A slots {g, g + 4}
//               (tcgen05.st, K-major A operand in TMEM; encoding checked by
//               tools/microbench/umma_tmem_a.cu)
//   warps 16-23 epilogue: tcgen05.ld 32x32b -> scaled, coalesced column
//               stores of U (two warps per TMEM lane quarter, alternate
//               16-column groups)
//   warps 24-25 loaders: fp32 chunk [16 columns][128 rows] by cp.async
//               (16 B per lane, a warp a whole 512-byte column segment)
//   warp 26     W pieces + scales (one bulk copy) + MMA issue (one thread)
// The encodings (descriptors, instruction descriptor, TMEM load shape) are
// the ones checked by tools/microbench/umma_test.cu on the B200.
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

#ifndef TM_LOAD_WARPS
#define TM_LOAD_WARPS 2  // loader warps (4 measured 5% slower)
#endif

namespace mpsvd {
namespace dev {
namespace tc {

constexpr int kBM = 128;                    // rows per tile = UMMA M
constexpr int kKC = 16;                     // K per chunk = UMMA K
constexpr int kStepCh = 2;  // chunks per pipeline step: one hand-off per 32 columns (c4 U 12.9 -> 11.9 ms)
constexpr int kStageBytes = kBM * kKC * kStepCh * 4;  // fp32 step: 16 KB
constexpr int kEpiWarps = 8;
constexpr int kSmemLimit = 227 * 1024;
constexpr int kHead = 14;                   // scaled operands stay below 2^14 (fp16 max 65504)

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
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(saddr(bar))
               : "memory");
}


// x = h + l, each an fp16 (the rounded remainder); packs 2 values per word
// (low half = the even K index).
__device__ __forceinline__ void split2h(float x0, float x1, uint32_t& h, uint32_t& l) {
  const __half2 bh = __floats2half2_rn(x0, x1);
  const float2 fh = __half22float2(bh);
  const __half2 bl = __floats2half2_rn(x0 - fh.x, x1 - fh.y);
  h = *reinterpret_cast<const uint32_t*>(&bh);
  l = *reinterpret_cast<const uint32_t*>(&bl);
}

// Byte offset of (mn, k) in an MN-major no-swizzle operand image whose MN
// extent is `mn_ext`: 8x8 core matrices of 128 B (mn contiguous, 16 B per k
// row), MN groups adjacent (SBO = 128 B), K groups `mn_ext/8 * 128` apart (LBO).
__host__ __device__ __forceinline__ uint32_t mn_major_off(int mn, int k, int mn_ext) {
  return (uint32_t)((((k >> 3) * (mn_ext >> 3) + (mn >> 3)) << 7) + ((k & 7) << 4) + ((mn & 7) << 1));
}

// W pieces + scales: [3 fp16 planes np x np][np floats 2^-s_c][np floats 2^t_j]
constexpr int kWPieces = 3;
__host__ __device__ __forceinline__ size_t wplanes_bytes(int np) {
  return (size_t)kWPieces * np * np * 2 + (size_t)2 * np * 4;
}

}  // namespace tc

// The Gram diagonal M_kk = ||a_k||^2, saved right after the Gram phase (the
// Jacobi then works on M in place) behind the W pieces and scales.
__global__ void av_tc_save_diag(const double* __restrict__ gram, int n, double* __restrict__ diag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) diag[k] = gram[(size_t)k * n + k];
}

// W (n x n, fp32, row-major rows of ldw = W^T buffer of finish_columns) and
// the saved Gram diagonal -> the three fp16 planes of 2^s_k W_kj 2^-t_j, each
// the np x np (K x N, N-major) smem image, and the column scales. One block
// per column j, thread = k.
__global__ void av_tc_prep_w(const float* __restrict__ w, int ldw, int n, int np, unsigned char* __restrict__ out,
                             const DevStatus* __restrict__ status) {
  const double* __restrict__ diag = reinterpret_cast<const double*>(out + tc::wplanes_bytes(np));
  if (status && status->status != kOk) return;
  __shared__ float red[4];
  const int j = blockIdx.x, k = threadIdx.x;
  int sk = 0;
  if (k < n) {
    const double d = diag[k];
    if (d > 0.0 && d <= 1.7976931348623157e308) {
      int e;
      frexp(sqrt(d), &e);  // ||a_k|| < 2^e
      sk = e - tc::kHead;
    }
  }
  const float x = (k < n && j < n) ? ldexpf(w[(long long)k * ldw + j], sk) : 0.0f;
  float mx = fabsf(x);
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((k & 31) == 0) red[k >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int i = 1; i < (int)((blockDim.x + 31) >> 5); ++i) mx = fmaxf(mx, red[i]);
  int tj = 0;
  if (mx > 0.0f && mx <= 3.4028235e38f) {
    int e;
    frexpf(mx, &e);  // max |2^s_k W_kj| < 2^e
    tj = e - tc::kHead;
  }
  if (k >= np) return;  // blockDim = max(np, 32): full warps for the shuffles
  const float xs = ldexpf(x, -tj);
  // w = w0 + w1 + w2 exactly (33 >= 24 bits) while w2 is a normal fp16, i.e.
  // for |xs| >= 2^8 (the column maximum is near 2^14); smaller entries keep
  // an absolute error below 2^-24 of the column maximum
  const __half w0 = __float2half_rn(xs);
  const float r1 = xs - __half2float(w0);
  const __half w1 = __float2half_rn(r1);
  const __half w2 = __float2half_rn(r1 - __half2float(w1));
  __half* planes = reinterpret_cast<__half*>(out);
  const uint32_t off = tc::mn_major_off(j, k, np) >> 1;  // in fp16 elements
  planes[off] = w0;
  planes[(size_t)np * np + off] = w1;
  planes[(size_t)2 * np * np + off] = w2;
  float* scl = reinterpret_cast<float*>(out + (size_t)tc::kWPieces * np * np * 2);
  if (j == 0) scl[k] = k < n ? ldexpf(1.0f, -sk) : 0.0f;
  if (k == 0) scl[np + j] = ldexpf(1.0f, tj);
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ void nbar_sync_k7(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

namespace tm {
#ifndef TM_GROUPS
#define TM_GROUPS 4  // converter groups (4 warps each); 2 left the MMA waiting for A slots (C4 ncu)
#endif
constexpr int kGroups = TM_GROUPS;
constexpr int kASlots = 2 * kGroups;  // TMEM A slots (16 columns each: 2 pieces x 8)
constexpr int kACols = tc::kStepCh * 2 * 8;  // per step: [chunk][piece][8 columns]
constexpr int kConvW = 4 * kGroups, kEpi0 = kConvW;  // converters: warps 0 .. kConvW-1, then 8 epilogue warps
constexpr int kLoad0 = kEpi0 + 8, kLoadWarps = TM_LOAD_WARPS, kMma = kLoad0 + kLoadWarps;
constexpr int kThreads = 32 * (kMma + 1);
constexpr int kPieces = 512 * 2 / (32 * kLoadWarps);  // 16-byte pieces per loader thread per step
}  // namespace tm

__global__ void __launch_bounds__(tm::kThreads, 1)
av_tc_tmem_f32(const float* __restrict__ a, long long lda, long long m, int n, int np,
               const unsigned char* __restrict__ wplanes, float* __restrict__ u, long long ldu,
               const DevStatus* __restrict__ status, int nstage, int acc_stride, int a_col0, int tcols) {
  using namespace tc;
  using namespace tm;
  if (status && status->status != kOk) return;
  extern __shared__ __align__(1024) unsigned char smem_tc[];
  const int nkc = (np + kKC * kStepCh - 1) / (kKC * kStepCh);  // steps per tile (the last may hold one chunk)
  const uint32_t wbytes = (uint32_t)wplanes_bytes(np);  // 3 fp16 W planes + A and U column scales
  const float* a_scl = reinterpret_cast<const float*>(smem_tc + (uint32_t)kWPieces * np * np * 2u);  // 2^-s_c per column of A
  const float* u_scl = a_scl + np;                                                    // 2^t_j per column of U
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
  const int kdbg = tcols >> 16;  // experiment switches (MPSVD_AV_DBG): 1 no MMA, 2 no U stores, 4 no split
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
        const int col = kc * kKC * kStepCh + c;
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
      // D f32, A fp16 K-major (TMEM), B fp16 MN-major (smem), N = np, M = 128
      const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | (1u << 16) | ((uint32_t)(np >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      const uint32_t w_lbo = (uint32_t)(np / 8) * 128;
      const uint32_t wbase = saddr(wsm);
      const uint32_t wplane = (uint32_t)np * np * 2u;
      // A1 W0 + A0 W2 + A0 W1 + A0 W0 (smallest first); A1 W1, A1 W2 (2^-22,
      // 2^-33 relative) are dropped
      const int pa[4] = {1, 0, 0, 0}, pw[4] = {0, 2, 1, 0};
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
          const int nsub = np - kc * kKC * kStepCh >= kKC * kStepCh ? kStepCh : 1;
          for (int h = 0; h < nsub; ++h) {
            const int kk = kc * kStepCh + h;  // 16-row K chunk of W
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (kdbg & 1) break;
              const uint64_t bd = umma_desc(wbase + (uint32_t)pw[q] * wplane + (uint32_t)kk * 2u * w_lbo, w_lbo, 128);
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                  "r"(at + (uint32_t)(h * 16 + pa[q] * 8)), "l"(bd), "r"(idesc), "r"((kk > 0 || q > 0) ? 1u : 0u));
            }
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
    mbar_wait(w_full, 0);  // the column scales arrive with the W pieces
    int slot = grp % nstage;
    unsigned sph = (unsigned)((grp / nstage) & 1);
    // one warp of the group polls each mbarrier, the other three wait on the
    // group's named barrier (all 16 converter warps polling took ~40% of the
    // SM's issue slots, ncu c4)
    for (int g = grp; g < nchunks; g += kGroups) {
      const int sl = g % kASlots;
      // the step's TMEM A slot must be free and its fp32 data present
      if (q == 0) {
        mbar_wait(&a_empty[sl], (unsigned)(((g / kASlots) & 1) ^ 1));
        mbar_wait(&stage_full[slot], sph);
      }
      nbar_sync_k7(1 + grp, 128);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const float* src = reinterpret_cast<const float*>(ssm + slot * kStageBytes);
      const int kc = g % nkc;
      const int nsub = np - kc * kKC * kStepCh >= kKC * kStepCh ? kStepCh : 1;
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a_col0 + sl * kACols);
      uint32_t dep = 0;
      for (int h = 0; h < nsub; ++h) {
        float v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = src[(h * kKC + c) * kBM + row];  // consecutive lanes: consecutive rows
        // column scales of these 16 columns (same address in every lane: broadcast)
        const float4* scl = reinterpret_cast<const float4*>(a_scl + (kc * kStepCh + h) * kKC);
        uint32_t hp[8], lp[8];
        if (kdbg & 4) {
#pragma unroll
          for (int c = 0; c < 8; ++c) hp[c] = lp[c] = __float_as_uint(v[2 * c]) ^ __float_as_uint(v[2 * c + 1]);
        } else {
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const float4 s4 = scl[c4];
            split2h(v[4 * c4] * s4.x, v[4 * c4 + 1] * s4.y, hp[2 * c4], lp[2 * c4]);
            split2h(v[4 * c4 + 2] * s4.z, v[4 * c4 + 3] * s4.w, hp[2 * c4 + 1], lp[2 * c4 + 1]);
          }
        }
        dep |= (lp[0] | lp[1] | lp[2] | lp[3]) | (lp[4] | lp[5] | lp[6] | lp[7]);
        const uint32_t th = ta + (uint32_t)(h * 16);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(th), "r"(hp[0]),
                     "r"(hp[1]), "r"(hp[2]), "r"(hp[3]), "r"(hp[4]), "r"(hp[5]), "r"(hp[6]), "r"(hp[7]));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(th + 8u),
                     "r"(lp[0]), "r"(lp[1]), "r"(lp[2]), "r"(lp[3]), "r"(lp[4]), "r"(lp[5]), "r"(lp[6]), "r"(lp[7]));
      }
      // release the staging slot only once every lane's loads have returned:
      // an arrive right after the loads (lane 0, after __syncwarp) can
      // overtake loads still in flight, and the loaders then overwrite the
      // slot under them (measured on K1z's identical ring, gram_ozaki32.cu
      // release_a). The arrive count depends on a warp OR-reduction of a
      // runtime zero derived from all loaded values (via the last pieces).
      {
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
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[sl]);
    }
  } else if (warp < tm::kEpi0 + kEpiWarps) {
    const int q = warp & 3, e = (warp - tm::kEpi0) >> 2;
    mbar_wait(w_full, 0);  // the column scales arrive with the W pieces
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
          // U_j = acc_j 2^t_j (exact: a power of two)
          const float4* us = reinterpret_cast<const float4*>(u_scl + c0);
          float x[16];
#pragma unroll
          for (int j4 = 0; j4 < 4; ++j4) {
            const float4 s4 = us[j4];
            x[4 * j4] = __uint_as_float(r[4 * j4]) * s4.x;
            x[4 * j4 + 1] = __uint_as_float(r[4 * j4 + 1]) * s4.y;
            x[4 * j4 + 2] = __uint_as_float(r[4 * j4 + 2]) * s4.z;
            x[4 * j4 + 3] = __uint_as_float(r[4 * j4 + 3]) * s4.w;
          }
          float* p = base + (long long)c0 * ldu;
          if (c0 + 16 <= n) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              *p = x[j];
              p += ldu;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c0 + j < n) p[(long long)j * ldu] = x[j];
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

// the pieces + scales, then the saved Gram diagonal (np doubles)
size_t av_tc_wplanes_bytes(int n) {
  const int np = (n + 15) / 16 * 16;
  return tc::wplanes_bytes(np) + (size_t)np * 8;
}

cudaError_t launch_av_tc_save_diag(const double* gram, int n, void* wplanes, cudaStream_t st) {
  const int np = (n + 15) / 16 * 16;
  av_tc_save_diag<<<(n + 127) / 128, 128, 0, st>>>(
      gram, n, reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(wplanes) + tc::wplanes_bytes(np)));
  return cudaGetLastError();
}

// experiment switches (MPSVD_AV_DBG): bit 0 skips the MMAs, bit 1 the U
// stores, bit 2 the split (c4, bf16x3 version: 14.8 ms; no MMA 11.1, no
// stores 12.8, no split 13.2, none of the three 8.1); MPSVD_AV_STAGES caps
// the staging ring (4-16 slots measured within 3%)
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
  if (prep)
    av_tc_prep_w<<<np, np < 32 ? 32 : np, 0, st>>>(w, ldw, n, np, reinterpret_cast<unsigned char*>(wplanes), status);
  const size_t wbytes = (wplanes_bytes(np) + 1023) & ~(size_t)1023;
  // accumulators [0, 2 acc_stride), A slots after them
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
  av_tc_tmem_f32<<<grid, tm::kThreads, smem, st>>>(a, lda, m, n, np, reinterpret_cast<const unsigned char*>(wplanes),
                                               u, ldu, status, nstage, acc_stride, a_col0,
                                               tcols | ((g_av_dbg & 7) << 16));
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace mpsvd
