// K2z: the double-double Gram M = A^T A of a binary64 A on the int8 tensor
// cores (Ozaki scheme), replacing K2's Dot2 loop on the fp64 pipe.
//
// Reference semantics: dd_gram (proj/tests/support/dd.cpp:75-88) - exact
// products, double-double accumulation - on the row-block plan of
// partitioned_gram (proj/src/parallel_gram.cpp:20-112). The result is not
// bit-identical to Dot2; it carries a normwise error far below the Dot2
// bound the tests hold K2 to (tests/test_ozaki.py).
//
// 1. ozaki_colexp: per row split s and column c, E[s][c] = the exponent with
//    max |a_kc| < 2^E over the split's rows (frexp of the column maximum).
// 2. ozaki_slice: every entry becomes the 88-bit fixed-point integer
//    X = trunc(x * 2^(86 - E)) (|X| < 2^86), written as 11 signed 8-bit
//    digits X = sum_p d_p 2^(8 (11 - p)), d_p in [-128, 127]: the bytes of
//    X + 0x80...80 (11 bytes), each XOR 0x80 (balanced digits, carries
//    resolved by the addition). Digit planes are stored as UMMA operand
//    images: [32-row chunk][digit][128-column block] x 4 KB, K-major,
//    no swizzle (8x16-byte core matrices; K neighbours 128 B apart, 8-row
//    groups 256 B apart), so the Gram kernel moves them with plain bulk copies.
// 3. gram_dd_ozaki: for a 128 x 128 output tile (I <= J), sum_k x_ki x_kj =
//    2^(E_i + E_j - 172) sum_{p,q} 2^(8 (22 - p - q)) sum_k d_p(x_ki) d_q(x_kj).
//    The digit products with p + q = w <= 12 are kept (66 of them; dropped
//    terms are below 2^-82 of |x_ki x_kj| per row); every product is an
//    exact int8 MMA (tcgen05.mma kind::i8, M = 128, N = 128, K = 32) into an
//    int32 TMEM accumulator per weight. TMEM holds four 128 x 128
//    accumulators, so the weight quads {12,11,10,9} {8,7,6,5} {4,3,2} are
//    dealt to CTAs, each quad's steps cut into ranges of <= 4 (6 sub-groups,
//    sub_group()). Step p of a quad streams A_p and B_{w_hi - p} (4 KB each)
//    into one ring slot (24 slots) and issuer W_k multiplies A_{p-k} by it
//    (weight w_hi - k); two loader warps and eight issuing warps (W_k x step
//    parity) share the steps — one issuing thread could not keep up with the
//    MMA: its wait / descriptor / commit chain took ~300 cycles per MMA.
//    Accumulators stay exact (|d_p d_q| <= 2^14, span x products per weight
//    per chunk < 4096 chunks) and are drained every span into the CTA's
//    double-double partial tile: V = sum_k acc_k 2^(8k) (exact in int64),
//    (hi, lo) = (fl(V), V - fl(V)), scaled by 2^(E_i + E_j + 4 - 8 w_hi),
//    added with dd_add; the drain warps then zero the accumulators (every MMA
//    accumulates, so MMA order across issuers is irrelevant).
//    Partials use K2's layout ([slot][64x64 tile pair][64x64] double2,
//    slot = split * 6 + sub-group), so the combine, the reference tree and
//    the multi-GPU exchange are K2's.
//
// Measured on B200 (tools/microbench/umma_i8.cu): an M128 K32 kind::i8 MMA
// takes 128 cycles at N = 256 and 64 at N = 128 when issued back to back
// (4.77 POPS over 148 SMs).
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace mpsvd {
namespace dev {
namespace oz {

constexpr int kL = 11;                 // digits per entry
constexpr int kKC = 32;                // rows per chunk = UMMA K (int8)
constexpr int kCB = 128;               // columns per digit block = UMMA M
constexpr int kPlane = kCB * kKC;      // 4096 bytes
constexpr int kGroups = 6;              // weight-quad x step-range sub-groups (sub_group)
constexpr int kBad = 1 << 20;          // E sentinel: the column holds inf/NaN
// Chunks per step: one slot, one wait and one release per kCPS MMAs (the
// per-MMA wait/commit chain bounded the first version: c3 Gram 25.5 ms at
// kCPS = 1, 20.6 at 2, 19.8 at 4; the issuers look back up to 3 slots, so
// the 192 KB ring keeps kRing = 6 slots at kCPS = 4)
constexpr int kCPS = 4;
constexpr int kRing = 6;               // step slots: kCPS A planes + kCPS B planes (4 KB each)
constexpr int kThreads = 448;          // warps 0-1 loaders, 2-5 drain, 6-13 MMA issuers (weight k, parity)

// Sub-group i: weight quad q ({12,11,10,9}, {8,7,6,5}, {4,3,2}: w_hi and
// nw weights w_hi - k, k < nw) and its steps [pa, pb] of 1..D (D = w_hi - 1),
// each quad's steps cut into ranges of at most 4 (6 sub-groups).
__host__ __device__ __forceinline__ void sub_group(int i, int& whi, int& nw, int& pa, int& pb) {
  for (int q = 0; q < 3; ++q) {
    const int h = 12 - 4 * q, d = h - 1, parts = (d + 3) / 4;
    if (i < parts) {
      const int base = d / parts, extra = d % parts;
      pa = 1 + i * base + (i < extra ? i : extra);
      pb = pa + base + (i < extra ? 1 : 0) - 1;
      whi = h;
      nw = q == 2 ? 3 : 4;
      return;
    }
    i -= parts;
  }
  whi = nw = pa = pb = 0;
}

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
__device__ __forceinline__ uint64_t kdesc(uint32_t addr) {  // K-major, no swizzle, LBO 128, SBO 256
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
// zero 16 TMEM columns of this warp's lane quarter
__device__ __forceinline__ void tmem_zero16(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(taddr),
      "r"(0u));
}
// Warp-converged issue: every lane runs the issuing loop (so its values stay
// in uniform registers) and only the leader lane's instruction is enabled.
__device__ __forceinline__ void umma_i8_lead(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc,
                                             uint32_t lead) {
  asm volatile(
      "{\n.reg .pred p, l;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 l, %5, 0;\n"
      "@l tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(lead));
}
__device__ __forceinline__ void umma_commit_lead(uint64_t* bar, uint32_t lead) {
  asm volatile(
      "{\n.reg .pred l;\nsetp.ne.b32 l, %1, 0;\n"
      "@l tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(saddr(bar)),
      "r"(lead)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_lead(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                              uint32_t lead) {
  asm volatile(
      "{\n.reg .pred l;\nsetp.ne.b32 l, %4, 0;\n"
      "@l mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n"
      "@l cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar)), "r"(lead)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_nox_lead(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                                  uint32_t lead) {
  asm volatile(
      "{\n.reg .pred l;\nsetp.ne.b32 l, %4, 0;\n"
      "@l cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar)), "r"(lead)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s2_lead(void* dst0, const void* src0, unsigned bytes0, void* dst1,
                                               const void* src1, unsigned bytes1, uint64_t* bar, uint32_t lead) {
  asm volatile(
      "{\n.reg .pred l;\nsetp.ne.b32 l, %7, 0;\n"
      "@l mbarrier.arrive.expect_tx.shared::cta.b64 _, [%6], %8;\n"
      "@l cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%6];\n"
      "@l cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%3], [%4], %5, [%6];\n}\n" ::"r"(
          saddr(dst0)),
      "l"(src0), "r"(bytes0), "r"(saddr(dst1)), "l"(src1), "r"(bytes1), "r"(saddr(bar)), "r"(lead),
      "r"(bytes0 + bytes1)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(saddr(bar))
               : "memory");
}

// X + 0x80..80 (11 bytes) as three words (bits 0-31, 32-63, 64-87) for
// X = sign(x) trunc(|x| 2^(86 - E)); requires |x| < 2^E.
__device__ __forceinline__ void fixed88(double x, int e_col, uint32_t& w0, uint32_t& w1, uint32_t& w2) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int e = (int)((bits >> 52) & 0x7ff);
  const unsigned long long mant = (bits & 0xFFFFFFFFFFFFFull) | (e ? (1ull << 52) : 0ull);
  const int s = (e ? e : 1) - 989 - e_col;  // |x| = mant 2^(e - 1075); X = mant 2^s, s <= 33
  unsigned long long lo = 0, hi = 0;
  if (s >= 0) {
    lo = mant << s;
    hi = s ? (mant >> (64 - s)) : 0ull;
  } else if (s > -64) {
    lo = mant >> (-s);
  }
  const unsigned long long olo = 0x8080808080808080ull, ohi = 0x808080ull;
  unsigned long long rlo, rhi;
  if ((long long)bits >= 0) {
    rlo = olo + lo;
    rhi = ohi + hi + (rlo < lo ? 1ull : 0ull);
  } else {
    rlo = olo - lo;
    rhi = ohi - hi - (olo < lo ? 1ull : 0ull);
  }
  w0 = (uint32_t)rlo;
  w1 = (uint32_t)(rlo >> 32);
  w2 = (uint32_t)rhi;
}

}  // namespace oz

// ---------------------------------------------------------------------------
// 1. column exponents per split: one warp per (split, column)
__global__ void __launch_bounds__(256)
ozaki_colexp(const double* __restrict__ a, long long lda, long long m, int n, const int* __restrict__ scb, int s0,
             int* __restrict__ e_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 8 + warp, s = s0 + blockIdx.y;
  if (c >= n) return;
  const long long r0 = (long long)scb[s] * oz::kKC;
  long long r1 = (long long)scb[s + 1] * oz::kKC;
  if (r1 > m) r1 = m;
  const double* col = a + (long long)c * lda;
  double mx = 0.0;
  bool bad = false;
  for (long long r = r0 + lane; r < r1; r += 128) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (r + 32 * u < r1) ? fabs(__ldg(col + r + 32 * u)) : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bad |= !(v[u] <= DBL_MAX);
      mx = fmax(mx, v[u]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, (int)bad, o) != 0;
  }
  if (lane == 0) {
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1): mx < 2^e
    e_out[(long long)s * n + c] = bad ? oz::kBad : e;
  }
}

// ---------------------------------------------------------------------------
// 2. digit planes: one (chunk, 128-column block) unit per iteration, 256
// threads = 128 columns x 2 row halves; A staged through shared memory with
// coalesced column reads.
// A tile = 128 columns x 32 rows of fp64, staged by cp.async (16 bytes per
// copy, 8 per thread) in a double buffer, so the next unit's loads are in
// flight while this one is split; column stride 34 doubles (16-byte aligned
// rows, 2-way bank conflicts at most on the reads).
__global__ void __launch_bounds__(256, 2)
ozaki_slice(const double* __restrict__ a, long long lda, long long m, int n, const int* __restrict__ e_cols,
            const int* __restrict__ scb, int nsplit, long long ch0, long long ch1, int ncb2,
            unsigned char* __restrict__ digits) {
  extern __shared__ __align__(16) double st_dyn[];
  constexpr int kLd = 34;
  const int tid = threadIdx.x;
  const int col = tid & 127, half = tid >> 7;
  const long long units = (ch1 - ch0) * ncb2;
  const bool aligned = (lda % 2 == 0) && (reinterpret_cast<uintptr_t>(a) % 16 == 0);
  // piece q = tid + 256 i (i < 8): column q >> 4, rows 2 (q & 15) .. + 1
  auto issue = [&](long long u, int buf) {
    const long long ch = ch0 + u / ncb2;
    const int cb = (int)(u % ncb2);
    const long long r0 = ch * oz::kKC;
    double* dst = st_dyn + buf * (oz::kCB * kLd);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int q = tid + 256 * i, c = q >> 4, rp = (q & 15) * 2;
      const int gc = cb * oz::kCB + c;
      const long long r = r0 + rp;
      // bytes present: 16 (both rows), 8 (the last row of an odd m) or 0; the rest is zero-filled
      const int bytes = gc < n && r < m ? (r + 1 < m ? 16 : 8) : 0;
      if (aligned) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + c * kLd + rp);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa),
                     "l"(bytes ? a + (long long)gc * lda + r : a), "r"(bytes)
                     : "memory");
      } else {  // odd lda or unaligned A: plain loads (visible after the __syncthreads)
        const double* sp = a + (long long)gc * lda + r;
        dst[c * kLd + rp] = bytes ? __ldg(sp) : 0.0;
        dst[c * kLd + rp + 1] = bytes == 16 ? __ldg(sp + 1) : 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  long long u = blockIdx.x;
  int buf = 0;
  if (u < units) issue(u, 0);
  for (; u < units; u += gridDim.x, buf ^= 1) {
    const long long un = u + gridDim.x;
    if (un < units) {
      issue(un, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const long long ch = ch0 + u / ncb2;
    const int cb = (int)(u % ncb2);
    // split of this chunk: last s with scb[s] <= ch
    int lo = 0, hi = nsplit - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (scb[mid] <= ch) lo = mid;
      else hi = mid - 1;
    }
    const int gc = cb * oz::kCB + col;
    const int e_col = gc < n ? e_cols[(long long)lo * n + gc] : 0;
    const double* src = st_dyn + buf * (oz::kCB * kLd) + col * kLd + 16 * half;
    uint32_t w[16][3];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      double x = src[r];
      if (e_col == oz::kBad) x = 0.0;
      oz::fixed88(x, e_col, w[r][0], w[r][1], w[r][2]);
    }
    unsigned char* base = digits + ((ch * oz::kL) * ncb2 + cb) * (long long)oz::kPlane + (col >> 3) * 256 +
                          half * 128 + (col & 7) * 16;
#pragma unroll
    for (int p = 1; p <= oz::kL; ++p) {
      const int b = oz::kL - p, wd = b >> 2, bb = b & 3;  // byte b of X' = digit p
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t t01 = __byte_perm(w[4 * j][wd], w[4 * j + 1][wd], bb | ((4 + bb) << 4));
        const uint32_t t23 = __byte_perm(w[4 * j + 2][wd], w[4 * j + 3][wd], bb | ((4 + bb) << 4));
        o[j] = __byte_perm(t01, t23, 0x5410) ^ 0x80808080u;
      }
      *reinterpret_cast<uint4*>(base + (long long)(p - 1) * ncb2 * oz::kPlane) = make_uint4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();  // this buffer is refilled by the next iteration's issue
  }
}

// ---------------------------------------------------------------------------
// 3. the Gram tiles: one CTA per (tile, sub-group, split), linear order
// tile fastest. Warps 0-1 load the steps (A plane + B plane, 4 KB each, per
// ring slot) of even / odd global step, warps 6-13 issue the MMAs (W_k x
// step parity), warps 2-5 drain (thread = tile row, tcgen05.ld 32x32b) into
// the double-double partial tile.
// MPSVD_OZAKI_PROF=1: per weight group, summed over CTAs: [0] CTAs, [1] MMA
// thread cycles, [2] of which waiting for planes, [3] waiting for the drain,
// [4] loader waiting for free slots, [5] drain cycles, [6] drain waiting
__device__ unsigned long long g_oz_prof[oz::kGroups][8];


__global__ void __launch_bounds__(oz::kThreads, 1)
gram_dd_ozaki(const unsigned char* __restrict__ digits, int ncb2, const int* __restrict__ e_cols, int n,
              const int2* __restrict__ tiles, const int* __restrict__ scb, int s0, int T64, int ntp64,
              double2* __restrict__ partials, int span_cap, int prof, int dbg, int ntiles, int ord) {
  using namespace oz;
  extern __shared__ __align__(1024) unsigned char smem_oz[];
  unsigned char* aring = smem_oz;
  unsigned char* bring = aring + kRing * kCPS * kPlane;
  uint64_t* bars = reinterpret_cast<uint64_t*>(bring + kRing * kCPS * kPlane);
  uint64_t* a_full = bars;  // one full barrier per step slot (A and B plane)
  uint64_t* a_empty = a_full + kRing;
  uint64_t* b_empty = a_empty + kRing;
  uint64_t* acc_full = b_empty + kRing;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  int* ej = reinterpret_cast<int*>(tmem_slot + 4);              // column exponents of block J

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // linear order: MPSVD_OZAKI_ORDER=1 sub-group fastest (the sub-groups of
  // one tile, which read the same two column blocks, run together), else
  // tile fastest; then split
  const unsigned inner = ord ? (unsigned)kGroups : (unsigned)ntiles;
  const unsigned a0 = blockIdx.x % inner, a1 = (blockIdx.x / inner) % (unsigned)(ntiles * kGroups / inner);
  const int tile = (int)(ord ? a1 : a0);
  const int g = (int)(ord ? a0 : a1);
  const int s = s0 + (int)(blockIdx.x / (unsigned)(ntiles * kGroups));
  const int2 ij = tiles[tile];  // (I, J): 128-column blocks, I <= J
  const int col0 = ij.y * kCB, ncol = kCB;
  int whi, nw, pa, pb;
  sub_group(g, whi, nw, pa, pb);
  const long long c0 = scb[s], c1 = scb[s + 1];
  // exact-accumulation span: chunks x products per weight per chunk < 4096
  // (|d_p d_q| <= 2^14, 32 rows per chunk: sums stay below 2^31)
  const int maxpairs = pb - pa + 1;
  int span = 1;
  while (span * 2 * maxpairs < 4096) span *= 2;
  if (span > span_cap) span = span_cap;
  const long long nspan = (c1 - c0 + span - 1) / span;
  const int npre = (pa - 1 < nw - 1) ? pa - 1 : nw - 1;  // leading A-only steps (A_{pa-npre} .. A_{pa-1})
  const int L = pb - pa + 1 + npre;                       // local steps per chunk

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], nw);
      mbar_init(&b_empty[i], nw);
    }
    mbar_init(acc_full, 2 * nw);
    mbar_init(acc_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp >= 2 && warp < 6) {
    for (int c = threadIdx.x - 64; c < kCB; c += 128) {
      const int gj = col0 + c;
      ej[c] = gj < n ? e_cols[(long long)s * n + gj] : 0;
    }
  }
  if (warp == 6) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(saddr(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  // Steps. Local step j of a chunk (global step t, slot t % kRing) covers
  // digit p = pa - npre + j: it brings A_p (block I) and, for p >= pa, B_q
  // with q = w_hi - p (block J). Issuer W_k (weight w_hi - k) multiplies
  // A_{p-k} (slot t - k) by B_q (slot t). Every issuer waits for both slots'
  // fills and then releases A of slot t - k and B of slot t at every step,
  // so each slot's empty barriers count nw arrivals per use and no release
  // can run ahead of the loader. Loaders and issuers split steps by the
  // parity of t; the integer accumulation makes MMA order irrelevant.
  if (warp < 2) {
    if (!(dbg & 1)) {
      const uint32_t lead = lane == 0;
      const unsigned par = (unsigned)warp;
      unsigned t = 0;
      unsigned long long tw = 0;
      // chunks grouped by kCPS inside each span (the issuers' grouping)
      for (long long cs = c0; cs < c1; cs += span) {
        const long long ce = cs + span < c1 ? cs + span : c1;
        for (long long ch = cs; ch < ce; ch += kCPS) {
          const int nc = (int)(ce - ch < kCPS ? ce - ch : kCPS);
          for (int j = 0; j < L; ++j, ++t) {
            if ((t & 1u) != par) continue;
            const int p = pa - npre + j;
            const int sl = (int)(t % kRing);
            const unsigned ph = ((t / kRing) & 1u) ^ 1u;
            const unsigned long long t0 = prof ? clock64() : 0;
            mbar_wait(&a_empty[sl], ph);
            mbar_wait(&b_empty[sl], ph);
            if (prof) tw += clock64() - t0;
            const unsigned bytes = (unsigned)nc * kPlane * (p < pa ? 1u : 2u);
            if (lead) mbar_expect_tx(&a_full[sl], bytes);
            for (int i = 0; i < nc; ++i) {
              const unsigned char* chunk = digits + ((ch + i) * kL) * ncb2 * (long long)kPlane;
              bulk_g2s_nox_lead(aring + ((size_t)sl * kCPS + i) * kPlane,
                                chunk + ((long long)(p - 1) * ncb2 + ij.x) * kPlane, kPlane, &a_full[sl], lead);
              if (p >= pa)
                bulk_g2s_nox_lead(bring + ((size_t)sl * kCPS + i) * kPlane,
                                  chunk + ((long long)(whi - p - 1) * ncb2 + ij.y) * kPlane, kPlane, &a_full[sl], lead);
            }
          }
        }
      }
      if (prof && lead && warp == 0) atomicAdd(&g_oz_prof[g][4], tw);
    }
  } else if (warp >= 6) {
    // issuers: warp 6 + 2k + par = W_k (weight w_hi - k) of the steps with t % 2 == par
    const int k = (warp - 6) >> 1;
    const unsigned par = (unsigned)((warp - 6) & 1);
    if (k < nw) {
      const uint32_t lead = lane == 0;
      // D s32, A s8, B s8, both K-major, N = 128, M = 128
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kCB >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      const uint32_t abase = saddr(aring), bbase = saddr(bring);
      const uint32_t dacc = tmem + (uint32_t)(k * kCB);
      unsigned t = 0;
      unsigned long long tacc = 0;
      const unsigned long long tstart = prof ? clock64() : 0;
      long long ch = c0;
      for (long long sp = 0; sp < nspan; ++sp) {
        const unsigned long long t0 = prof ? clock64() : 0;
        mbar_wait(acc_empty, (unsigned)(sp & 1));
        if (prof) tacc += clock64() - t0;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        long long ce = ch + span;
        if (ce > c1) ce = c1;
        for (; ch < ce; ch += kCPS) {
          const int nc = (int)(ce - ch < kCPS ? ce - ch : kCPS);
          for (int j = 0; j < L; ++j, ++t) {
            if ((t & 1u) != par) continue;
            const int p = pa - npre + j;
            const int sl = (int)(t % kRing);
            if (!(dbg & 1)) mbar_wait(&a_full[sl], (t / kRing) & 1u);
            const bool has_a = t >= (unsigned)k;
            const int sla = (int)((t + kRing - (unsigned)k) % kRing);
            if (has_a && k > 0 && !(dbg & 1)) mbar_wait(&a_full[sla], ((t - (unsigned)k) / kRing) & 1u);
            if (p >= pa && p - k >= 1) {
              asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
              for (int i = 0; i < nc; ++i)  // the group's chunks: the same weight, summed exactly
                umma_i8_lead(dacc, kdesc(abase + ((uint32_t)sla * kCPS + i) * kPlane),
                             kdesc(bbase + ((uint32_t)sl * kCPS + i) * kPlane), idesc, 1u, lead && !(dbg & 2));
            }
            if (!(dbg & 8)) {
              if (has_a) umma_commit_lead(&a_empty[sla], lead);
              umma_commit_lead(&b_empty[sl], lead);
            }
          }
        }
        umma_commit_lead(acc_full, lead);
      }
      if (prof && lead && k == 0 && par == 0) {
        atomicAdd(&g_oz_prof[g][0], 1ull);
        atomicAdd(&g_oz_prof[g][1], clock64() - tstart);
        atomicAdd(&g_oz_prof[g][3], tacc);
      }
    }
  } else if (warp < 6) {
    // drain: TMEM lane quarter q = warp % 4, thread = tile row
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int gi = ij.x * kCB + r;
    const int ei = gi < n ? e_cols[(long long)s * n + gi] : 0;
    const int ti = gi >> 6;
    const long long slot = (long long)s * kGroups + g;
    auto out_ptr = [&](int c) -> double2* {
      const int gj = col0 + c, tj = gj >> 6;
      if (c >= ncol) return nullptr;
      if (ti > tj || tj >= T64) return nullptr;
      const int tp = ti * T64 - (ti * (ti - 1)) / 2 + (tj - ti);
      return partials + (slot * ntp64 + tp) * 4096 + (gi & 63) * 64 + (gj & 63);
    };
    if (nspan == 0) {
      for (int c = 0; c < ncol; ++c) {
        double2* o = out_ptr(c);
        if (o) *o = make_double2(0.0, 0.0);
      }
    }
    // accumulators start at zero; every MMA accumulates
    for (int c = 0; c < 512; c += 16) tmem_zero16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c);
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(acc_empty);
    unsigned long long tdr = 0, tdw = 0;
    for (long long sp = 0; sp < nspan; ++sp) {
      const unsigned long long t0 = prof ? clock64() : 0;
      mbar_wait(acc_full, (unsigned)(sp & 1));
      const unsigned long long t1 = prof ? clock64() : 0;
      tdw += t1 - t0;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      for (int c0 = 0; c0 < ncol; c0 += 8) {
        uint32_t v[4][8];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k < nw)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                         : "=r"(v[k][0]), "=r"(v[k][1]), "=r"(v[k][2]), "=r"(v[k][3]), "=r"(v[k][4]), "=r"(v[k][5]),
                           "=r"(v[k][6]), "=r"(v[k][7])
                         : "r"(taddr + (uint32_t)(k * kCB)));
          else
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) v[k][jj] = 0u;
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(
                           taddr + (uint32_t)(k * kCB)),
                       "r"(0u));
        // the running partials of the 16 columns are loaded together (one
        // memory latency per group, not per entry)
        double2* op[8];
        double2 old[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          op[jj] = out_ptr(c0 + jj);
          old[jj] = (sp > 0 && op[jj]) ? *op[jj] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int c = c0 + jj;
          double2* o = op[jj];
          if (!o) continue;
          // acc k holds weight w_hi - k, worth 2^(8k) of weight w_hi: exact in int64
          const long long vv = (long long)(int)v[0][jj] + (long long)(int)v[1][jj] * 256 +
                               (long long)(int)v[2][jj] * 65536 + (long long)(int)v[3][jj] * 16777216;
          const double hi = (double)vv;
          const double lo = (double)(vv - (long long)hi);
          const int e2 = ej[c];
          dd t;
          if (ei == kBad || e2 == kBad) {
            t = dd_make(__longlong_as_double(0x7ff8000000000000ll), 0.0);
          } else {
            const int sc = ei + e2 + 4 - 8 * whi;
            t = dd_make(scalbn(hi, sc), scalbn(lo, sc));
          }
          if (sp > 0) t = dd_add(dd_make(old[jj].x, old[jj].y), t);
          *o = make_double2(t.hi, t.lo);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      if (prof) tdr += clock64() - t1;
    }
    if (prof && warp == 2 && lane == 0) {
      atomicAdd(&g_oz_prof[g][5], tdr);
      atomicAdd(&g_oz_prof[g][6], tdw);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 6) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

// ---------------------------------------------------------------------------
size_t ozaki_digit_bytes(long long m, int n) {
  const long long nch = (m + oz::kKC - 1) / oz::kKC;
  const long long ncb2 = ((n + 255) / 256) * 2;
  return (size_t)nch * oz::kL * ncb2 * oz::kPlane;
}
int ozaki_groups() { return oz::kGroups; }

// Tiles (I, J) of 128-column blocks with I <= J (the upper triangle)
void ozaki_tiles(int n, std::vector<int2>& tiles) {
  tiles.clear();
  const int T = (n + 127) / 128;
  for (int J = 0; J < T; ++J)
    for (int I = 0; I <= J; ++I) tiles.push_back(make_int2(I, J));
}

static size_t ozaki_smem() {
  return (size_t)oz::kRing * 2 * oz::kCPS * oz::kPlane + 3 * oz::kRing * 8 + 16 + 16 + 128 * 4 + 64;
}

cudaError_t launch_gram_ozaki(const double* a, long long lda, long long m, int n, const int* scb_dev,
                              const int* scb_host, int nsplit_total, int s0, int ns, const int2* tiles, int ntiles,
                              int* e_cols, unsigned char* digits, double2* partials, int ntp64, int sm_count,
                              cudaStream_t st) {
  if (ns <= 0) return cudaSuccess;
  const int T64 = (n + 63) / 64;
  const int ncb2 = ((n + 255) / 256) * 2;
  // test hook: chunks per exact-accumulation span (read per launch)
  const char* span_env = getenv("MPSVD_OZAKI_SPAN");
  const int span_cap = span_env && atoi(span_env) > 0 ? atoi(span_env) : 1 << 20;
  dim3 gce((n + 7) / 8, ns);
  ozaki_colexp<<<gce, 256, 0, st>>>(a, lda, m, n, scb_dev, s0, e_cols);
  const long long ch0 = scb_host[s0], ch1 = scb_host[s0 + ns];
  const long long units = (ch1 - ch0) * ncb2;
  if (units > 0) {
    // per-device attribute: set on every launch (a process may drive several GPUs)
    cudaError_t e = cudaFuncSetAttribute(ozaki_slice, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(2 * oz::kCB * 34 * sizeof(double)));
    if (e != cudaSuccess) return e;
    long long grid = units < (long long)sm_count * 2 ? units : (long long)sm_count * 2;
    ozaki_slice<<<(int)grid, 256, 2 * oz::kCB * 34 * sizeof(double), st>>>(a, lda, m, n, e_cols, scb_dev,
                                                                           nsplit_total, ch0, ch1, ncb2, digits);
  }
  const size_t smem = ozaki_smem();
  {
    cudaError_t e = cudaFuncSetAttribute(gram_dd_ozaki, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const char* prof_env = getenv("MPSVD_OZAKI_PROF");
  const int prof = prof_env && prof_env[0] == '1';
  const char* dbg_env = getenv("MPSVD_OZAKI_DBG");  // bit 0: no plane loads, bit 1: no MMAs, bit 3: no releases
  // (timing probes; bit 3 only together with bit 0)
  const int dbg = dbg_env ? atoi(dbg_env) : 0;
  if (prof) {
    unsigned long long z[oz::kGroups * 8] = {};
    cudaMemcpyToSymbolAsync(g_oz_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
  }
  const char* ord_env = getenv("MPSVD_OZAKI_ORDER");
  const int ord = ord_env ? atoi(ord_env) : 0;
  const unsigned grid = (unsigned)(ntiles * oz::kGroups * ns);
  gram_dd_ozaki<<<grid, oz::kThreads, smem, st>>>(digits, ncb2, e_cols, n, tiles, scb_dev, s0, T64, ntp64, partials,
                                                  span_cap, prof, dbg, ntiles, ord);
  if (prof) {
    unsigned long long h[oz::kGroups * 8];
    cudaMemcpyFromSymbolAsync(h, g_oz_prof, sizeof(h), 0, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    for (int g = 0; g < oz::kGroups; ++g) {
      const double c = h[g * 8] ? (double)h[g * 8] : 1.0;
      fprintf(stderr,
              "ozaki prof g%d: CTAs %llu | per CTA (kcycles): mma %.1f (plane wait %.1f, drain wait %.1f) loader "
              "slot wait %.1f | drain %.1f (acc wait %.1f)\n",
              g, h[g * 8], h[g * 8 + 1] / c / 1e3, h[g * 8 + 2] / c / 1e3, h[g * 8 + 3] / c / 1e3, h[g * 8 + 4] / c / 1e3,
              h[g * 8 + 5] / c / 1e3, h[g * 8 + 6] / c / 1e3);
    }
  }
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace mpsvd
