// K1z: the binary64 Gram M = A^T A of a binary32 A (n <= 128) on the int8
// tensor cores (Ozaki scheme), the fp32 sibling of K2z (gram_ozaki.cu).
//
// Reference semantics: partitioned_gram of cast(A, Higher) (proj/src/
// parallel_gram.cpp:79-112, thinsvd.cpp:61-70): exact binary32 -> binary64
// widening, exact products, binary64 accumulation in a fixed order, exactly
// symmetric result. Any fixed summation order is allowed; the
// acceptance criterion is ||dM||_F / ||M||_F <= 10 m u_h
// (proj/tests/test_parallel_gram.cpp:74-86). K1z replaces the binary64
// accumulation by an exact integer one: every entry is truncated once to a
// 47-bit fixed-point grid of its column (below), the digit products are
// summed exactly, and each CTA's span totals are carried in double-double;
// the result is rounded to binary64 once. DESIGN.md §3 gives the error
// analysis; tests/test_ozaki32.py pins it bitwise to the C restatement
// (oracle/mpsvd_port.c port_gram_f32_ozaki) and to the reference criterion.
//
// Work split. The rows are cut into 32-row chunks (the kind::i8 UMMA K) and
// the pipeline moves 64-row steps (two chunks). A launch covers a chunk
// range; CTA pair p (a cluster of 2) takes an equal share of it, CTA g of
// the pair owns accumulator group g (below) and loads, scans and converts
// chunk 2j + g of step j; the two chunks meet in both CTAs' digit slots.
// Per CTA:
//   warp 0       TMA: this CTA's chunk of each step (32 rows x 128 columns,
//                16 KB, 128B swizzle) into a ring
//   warp 1       MMA issue (one thread, 12 products per step as 10 / 8 MMAs)
//                + TMEM allocation
//                (4 x 128 columns); in group 1 the warp also sums the D8
//                diagonal (below)
//   warps 2-5    drain (TMEM lane quarter = tile rows): span totals -> dd
//   warps 6-21   convert, two groups of 8 warps taking alternate steps;
//                thread = (column, 16 rows): the 6 signed digits of every
//                entry as UMMA operand planes (K-major, no swizzle) in this
//                CTA's half (two 16-row K-core groups) of a digit slot
//   warps 22-25  scouts: lane = column; the column maxima of this CTA's
//                chunk, exchanged with the peer's (st.async into its smem,
//                completing on an mbarrier) -> the step's maxima -> the span
//                decision (one 128-thread barrier-with-reduction) and the
//                span's exponents, published per step by an mbarrier
//   warp 26      copier: one DSMEM bulk copy (24 KB) moves this CTA's half
//                of each digit slot into the peer's slot (transaction bytes
//                on the peer's slot barrier), so each row is converted once
// A slot is released by the warps that read it only once every lane's loads
// have returned (release_a: a plain lane-0 arrive after __syncwarp let the
// TMA refill a slot under loads still in flight, tools/oz32_harness.cu).
// Per role one warp polls an mbarrier and the role's other warps wait on a
// named barrier. The per-step hand-off chain (TMA -> scouts -> converter
// group -> DSMEM copy -> MMA -> multicast release) paces the kernel: with
// MMAs, conversion and the scouts' exchange all skipped (MPSVD_OZ32_DBG) a
// 32-row step still took ~1,000 cycles, so the step was doubled to 64 rows
// (c4 Gram 22.5 -> 17.3 ms).
//
// Digits. A span is a run of steps with fixed column exponents E_c. A span
// starts at the first step of the pair's range, after kSpanMax steps (the
// int32 accumulators stay exact), or at a step holding an entry with
// |x| >= 2^E_c; it sets E_c = e(colmax of that step) + kHead (frexp
// exponent, colmax < 2^e), or kZeroE for an all-zero column. Within the span
// every x of column c becomes X = sign(x) round(|x| 2^(46 - E_c)),
// |X| < 2^46, written as 6 balanced digits X = sum_p d_p 2^(8 (6 - p)),
// d_p in [-128, 127]: the bytes of X + 0x808080808080, each XOR 0x80.
// Products. x_ki x_kj ~ 2^(E_i + E_j - 92) sum_{p,q} d_p d_q 2^(8 (12 - p - q));
// the weights s = p + q <= 7 are kept. The tile is diagonal (n <= 128), so
// S_s = sum_{p+q=s} A_p^T A_q = T_s + T_s^T + D_s with T_s = sum_{p<q} and
// D_s = A_{s/2}^T A_{s/2}: 12 products per chunk instead of 21, in 8
// accumulators, which TMEM (512 columns) holds 4 at a time - hence the CTA
// pair: group 0 = {T7: (1,6)(2,5)(3,4), T3: (1,2), T4: (1,3), D2: (1,1)},
// group 1 = {T5: (1,4)(2,3), T6: (1,5)(2,4), D4: (2,2), D6: (3,3)},
// 6 products (M = N = 128, K = 32, 64 cycles each) per chunk per CTA, issued
// as 5 / 4 MMAs (adjacent B planes merged into N = 256, issue_chunk). Of the
// dropped weights only D8 = A_4^T A_4 has a non-zero mean (on the diagonal,
// sum_k d_4(x_ki)^2 >= 0); its diagonal is summed on the CUDA cores by the
// MMA warp of group 1 (dp4a on plane 4) and added to M_ii by its drain. Every
// other dropped term is zero-mean noise of ~2^-39 colmax_i colmax_j per row.
// Drain. At a span end every entry's group total is formed exactly
// (int64 / double pieces), scaled by 2^(E_i + E_j - 92 + ...) - D terms
// with an extra 1/2, so that M = P + P^T - and dd_add-ed into the CTA's
// double-double partial P (stored [j][i], i contiguous). A final kernel adds
// the partials of every CTA (fixed order: P(i,j) then P(j,i)) and rounds
// once to binary64, writing both triangles. Columns holding inf / NaN give
// NaN in their row and column of M.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace mpsvd {
namespace dev {
namespace oz32 {

constexpr int kKC = 32;                       // rows per chunk = UMMA K (int8)
constexpr int kCB = 128;                      // tile columns = UMMA M = N
constexpr int kPlane = kCB * kKC;             // 4096 bytes per digit plane
constexpr int kDigits = 6;
constexpr int kHead = 2;                      // exponent headroom (bits) of a new span
constexpr int kSpanMax = 512;                 // steps (2 chunks) per span: int32 sums stay exact
constexpr int kZeroE = -160;                  // exponent of an all-zero column
// The pipeline moves 64-row steps (two chunks): CTA g of the pair loads,
// scans and converts chunk 2j + g of step j; the peer's chunk arrives by one
// DSMEM copy; both CTAs run 12 MMAs per step.
constexpr int kStep = 2;                          // chunks per step
constexpr int kAStageBytes = kKC * kCB * 4;       // 16384: this CTA's chunk, 128 columns x 128 B, 128B-swizzled
constexpr int kPmaxSlots = 16;                // ring of the peer's half-chunk column maxima (> A + digit slots)
constexpr int kConvGroups = 2;                // converter groups: group G converts the chunks j = G mod 2
constexpr int kConvThreads = 256 * kConvGroups;
constexpr int kConvWarp0 = 6;
constexpr int kScoutWarp0 = kConvWarp0 + kConvThreads / 32, kScoutWarps = 4;
constexpr int kWarpCopy = kScoutWarp0 + kScoutWarps;  // DSMEM bulk copies of this CTA's digit half to the peer
constexpr int kThreads = 32 * (kWarpCopy + 1);
constexpr int kGroupWarps = 8;                // converter warps per group (one chunk half: 128 columns x 2)
constexpr int kHalfBytes = kDigits * 2048;    // one 16-row K-core group of a digit slot: 6 planes x 2 KB
constexpr int kDStageBytes = 2 * kStep * kHalfBytes;  // a step's 4 K-core groups (64 rows) x 6 planes
constexpr unsigned long long kC48 = 0x808080808080ull;

// frexp exponent of a non-negative finite binary32 bit pattern (v < 2^e), or
// -1000 for zero
__host__ __device__ __forceinline__ int fexp_bits(uint32_t ab) {
  const int e8 = (int)(ab >> 23);
  if (e8) return e8 - 126;
  if (!ab) return -1000;
#ifdef __CUDA_ARCH__
  return (32 - __clz((int)ab)) - 149;
#else
  return (32 - __builtin_clz(ab)) - 149;
#endif
}

// X + 0x808080808080 for X = RNE(x 2^(46 - E)) (round to nearest, ties to
// even), |x| < 2^E: rounding, not truncation, so the grid error has zero
// mean and the diagonal of M carries no bias. Exact integer form (the
// converters' path for columns with E < -78, and the restatement's).
__host__ __device__ __forceinline__ unsigned long long fixed48(uint32_t b, int E) {
  const uint32_t e8 = (b >> 23) & 0xFFu;
  if (e8 == 0xFFu) return kC48;  // inf / NaN: handled as a flagged zero
  const uint32_t mant = (b & 0x7FFFFFu) | (e8 ? 0x800000u : 0u);
  const int sh = (int)(e8 ? e8 : 1u) - 104 - E;
  unsigned long long X = 0;
  if (mant) {
    if (sh >= 0) {
      X = (unsigned long long)mant << sh;
    } else if (sh > -64) {
      const int s = -sh;
      const unsigned long long r = (unsigned long long)mant >> s;
      const unsigned long long rem = (unsigned long long)mant - (r << s), half = 1ull << (s - 1);
      X = r + ((rem > half || (rem == half && (r & 1ull))) ? 1ull : 0ull);
    }
  }
  return (b >> 31) ? kC48 - X : kC48 + X;
}

// The same on the fp64 pipe, for columns with E >= -78 (or all-zero, E_f = 0
// then): the binary32 bits re-biased into a binary64 scaled by 2^(46 - E)
// (exact), plus 1.5 2^52 + 0x808080808080 - the sum has ulp 1, so it rounds
// the scaled value to the nearest integer, ties to even (the constant is
// even), and its low 48 bits are X + 0x808080808080. Zero and subnormal x
// become 2^(-81-E) (1 + f) < 1/2 and round to 0, as the exact form gives.
// kc = (942 - E) << 20.
__device__ __forceinline__ void fixed48_fast(uint32_t b, uint32_t kc, uint32_t& lo, uint32_t& hi) {
  const uint32_t h = (((b >> 3) & 0x0FFFFFFFu) + kc) | (b & 0x80000000u);
  const double d = __hiloint2double((int)h, (int)(b << 29));
  const double w = __dadd_rn(d, 6755399441055744.0 + 141289400074368.0);  // 1.5 2^52 + 0x808080808080
  lo = (uint32_t)__double2loint(w);
  hi = (uint32_t)__double2hiint(w);
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
// try_wait with a long suspend-time hint (wait mode 0). The hinted sleep
// ends at any mbarrier activity of the CTA, so in this kernel (barriers
// updated every few cycles) a waiting warp re-polls every ~20 ns: the drain
// warps' span-long waits alone took 18% of all issue slots (ncu, c4). Wait
// mode 2 polls once and then backs off by a per-site __nanosleep, long for
// the waits that span many chunks (drain, accumulator hand-off), short or
// none on the per-chunk hand-offs.
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(saddr(b)), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, unsigned parity) {
  uint32_t done;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(saddr(b)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, unsigned parity) {
  uint32_t done;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(saddr(b)), "r"(parity)
      : "memory");
  return done != 0;
}
// Release an A slot after this warp's shared-memory loads of it (called by
// every lane; dep = the lane's loaded data). The arrive must not overtake a
// load still in flight, or the TMA refills the slot under it: measured, with
// 4-7 A slots and a plain lane-0 arrive after __syncwarp, the converters'
// second LDS of a chunk sometimes returned the next occupant's data
// (tools/oz32_harness.cu). A zero derived from every lane's loaded registers
// is OR-reduced over the warp (REDUX waits for all lanes' loads to return)
// and lane 0's arrive count depends on it.
// zmask is a runtime zero (a kernel argument's unused bits): ptxas folds an
// AND with the constant 0 and the dependency with it.
__device__ __forceinline__ void release_a(uint64_t* b, int lane, uint32_t dep, uint32_t zmask) {
  uint32_t z = __reduce_or_sync(0xffffffffu, dep & zmask);
  if (lane == 0)
    asm volatile(
        "{\n.reg .b32 cnt;\nadd.u32 cnt, %1, 1;\n"
        "mbarrier.arrive.shared::cta.b64 _, [%0], cnt;\n}\n" ::"r"(saddr(b)),
        "r"(z)
        : "memory");
}
// cluster-scope acquire (the digit slots are also filled by the peer CTA's
// converters, which arrive with release.cluster)
__device__ __forceinline__ void mbar_wait_cl(uint64_t* b, unsigned parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_v2(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
// named barrier (hardware wait, no issue slots): one warp of a role polls the
// mbarrier, the role's other warps block here until it has seen the phase
__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// MMA completion -> the mbarrier at this offset in both CTAs of the pair,
// issued only after `dep` (a runtime zero derived from loads that must have
// returned first) is available
__device__ __forceinline__ void commit_lead_pair_dep(uint64_t* bar, uint32_t lead, uint32_t dep) {
  asm volatile(
      "{\n.reg .pred l;\nsetp.ne.b32 l, %1, 0;\n"
      "@l tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %2;\n}\n" ::
          "r"(saddr(bar) + dep),
      "r"(lead), "h"((unsigned short)3)
      : "memory");
}
// MMA completion -> the mbarrier at this offset in both CTAs of the pair
__device__ __forceinline__ void commit_lead_pair(uint64_t* bar, uint32_t lead) {
  asm volatile(
      "{\n.reg .pred l;\nsetp.ne.b32 l, %1, 0;\n"
      "@l tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %2;\n}\n" ::
          "r"(saddr(bar)),
      "r"(lead), "h"((unsigned short)3)
      : "memory");
}
// wmode 0: hinted try_wait; 1: un-hinted try_wait loop; 2: test_wait with
// __nanosleep(ns) back-off (ns = 0: un-hinted try_wait loop)
__device__ __forceinline__ void mbar_wait_m(uint64_t* b, unsigned parity, int wmode, unsigned ns) {
  if (wmode == 0) {
    mbar_wait(b, parity);
  } else if (wmode == 1 || ns == 0) {
    while (!mbar_try(b, parity)) {
    }
  } else {
    while (!mbar_test(b, parity)) __nanosleep(ns);
  }
}
// Digit slot layout: [K half h][digit p][16 column groups][8 columns x 16 B],
// i.e. K-major, no swizzle, with the two 16-row K halves kHalfBytes apart
// (LBO) and 8-column groups 128 B apart (SBO): each CTA's half of a slot is
// one contiguous block, moved to the peer by a single bulk copy.
__device__ __forceinline__ uint64_t kdesc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(kHalfBytes >> 4) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void bulk_s2peer(uint32_t dst_cl, uint32_t src, unsigned bytes, uint32_t bar_cl) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   dst_cl),
               "r"(src), "r"(bytes), "r"(bar_cl)
               : "memory");
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(saddr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(saddr(bar))
      : "memory");
}

__device__ __forceinline__ void umma_i8_lead(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc,
                                             uint32_t lead) {
  asm volatile(
      "{\n.reg .pred p, l;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 l, %5, 0;\n"
      "@l tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(lead));
}
__device__ __forceinline__ void commit_lead(uint64_t* bar, uint32_t lead) {
  asm volatile(
      "{\n.reg .pred l;\nsetp.ne.b32 l, %1, 0;\n"
      "@l tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(saddr(bar)),
      "r"(lead)
      : "memory");
}
__device__ __forceinline__ void arrive_lead(uint64_t* bar, uint32_t lead) {
  asm volatile(
      "{\n.reg .pred l;\nsetp.ne.b32 l, %1, 0;\n"
      "@l mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::"r"(saddr(bar)),
      "r"(lead)
      : "memory");
}
// The MMAs of one chunk for group G: operand descriptors are the slot's
// base descriptor plus the plane offset >> 4. Digit planes q and q + 1 are
// contiguous along N (16 + 16 eight-column groups, 128 B apart), so two
// products with the same A plane and adjacent B planes are ONE N = 256 MMA
// into two adjacent accumulators (the A plane is read once: 5 / 4 MMAs per
// chunk instead of 6, 44 / 40 KB of operands instead of 48). Accumulator
// columns (128 each):
//   group 0: T7 (1,6)(2,5)(3,4) -> 0, [T3 | T4] = A_1^T [A_2 | A_3] -> 1, 2, D2 (1,1) -> 3
//   group 1: [T5 | T6] = A_1^T [A_4 | A_5] + A_2^T [A_3 | A_4] -> 0, 1, D4 (2,2) -> 2, D6 (3,3) -> 3
// idesc = N = 128, idesc2 = N = 256. The restatement (oracle/mpsvd_port.c
// o32_product) lists the same twelve products one by one; the sums are exact
// integers, so the grouping cannot change a bit.
template <int G>
__device__ __forceinline__ void issue_chunk(uint32_t tmem, uint64_t sd, uint32_t idesc, uint32_t idesc2, bool fresh,
                                            uint32_t lead) {
  const uint32_t acc0 = fresh ? 0u : 1u;
#define OZ32_PL(p) (sd + (uint64_t)(((p) - 1) * (2048 >> 4)))
  if (G == 0) {
    umma_i8_lead(tmem, OZ32_PL(1), OZ32_PL(6), idesc, acc0, lead);
    umma_i8_lead(tmem, OZ32_PL(2), OZ32_PL(5), idesc, 1u, lead);
    umma_i8_lead(tmem, OZ32_PL(3), OZ32_PL(4), idesc, 1u, lead);
    umma_i8_lead(tmem + (uint32_t)kCB, OZ32_PL(1), OZ32_PL(2), idesc2, acc0, lead);
    umma_i8_lead(tmem + (uint32_t)(3 * kCB), OZ32_PL(1), OZ32_PL(1), idesc, acc0, lead);
  } else {
    umma_i8_lead(tmem, OZ32_PL(1), OZ32_PL(4), idesc2, acc0, lead);
    umma_i8_lead(tmem, OZ32_PL(2), OZ32_PL(3), idesc2, 1u, lead);
    umma_i8_lead(tmem + (uint32_t)(2 * kCB), OZ32_PL(2), OZ32_PL(2), idesc, acc0, lead);
    umma_i8_lead(tmem + (uint32_t)(3 * kCB), OZ32_PL(3), OZ32_PL(3), idesc, acc0, lead);
  }
#undef OZ32_PL
}

// Exact group total of one tile entry from the 4 accumulators, relative to
// 2^(base) with base = 40 (group 0) or 47 (group 1), as a double-double.
__device__ __forceinline__ dd group_total(int g, int a0, int a1, int a2, int a3) {
  if (g == 0) {
    // T7 * 2^0 + T4 * 2^24 + (T3 * 2^32 + D2 * 2^39), D2 already halved (2^40 -> 2^39)
    const long long vlo = (long long)a0 + (long long)a1 * 16777216LL;          // |.| < 2^56
    const long long vhi = (long long)a2 + (long long)a3 * 128LL;               // |.| < 2^39
    const double lh = (double)vlo;
    const double ll = (double)(vlo - (long long)lh);
    return dd_add(dd_make((double)vhi * 4294967296.0, 0.0), dd_make(lh, ll));
  }
  // T6 * 2^1 + T5 * 2^9 + D4 * 2^16 + D6 * 2^0 (D4, D6 halved): |.| < 2^48, exact
  const long long v = (long long)a0 * 2LL + (long long)a1 * 512LL + (long long)a2 * 65536LL + (long long)a3;
  return dd_make((double)v, 0.0);
}

}  // namespace oz32

using namespace oz32;

// Debug hook, compiled only with -DOZ32_DEBUG (tools/oz32_harness.cu): per
// global chunk, the digits the converters wrote ([chunk][digit][column][32
// rows] int8), the exponent each column used, the MMA's span-start flag and
// per-stage clock64 stamps of pair 0.
#ifdef OZ32_DEBUG
struct Oz32Dbg {
  int8_t* digits;
  short* E;
  int* fresh;
  unsigned long long* prof;  // [cta 0/1 of pair 0][chunk][12] clock64 stamps
  int prof_chunks;
};
__device__ Oz32Dbg g_oz32_dbg = {nullptr, nullptr, nullptr, nullptr, 0};
__device__ __forceinline__ void oz32_stamp(const Oz32Dbg& d, int g, int pair, int j, int ev) {
  if (d.prof && pair == 0 && j < d.prof_chunks) d.prof[((size_t)g * d.prof_chunks + j) * 12 + ev] = clock64();
}
#define OZ32_DBG(...) __VA_ARGS__
#else
#define OZ32_DBG(...)
#endif

// ---------------------------------------------------------------------------
template <int kAStages, int kDStages>
__global__ void __launch_bounds__(kThreads, 1)
gram_f32_ozaki(const __grid_constant__ CUtensorMap amap, int n, long long c_begin, long long c_end, int npairs,
               double2* __restrict__ partials, int* __restrict__ bad_cols, int accumulate, int span_max, int wmode) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-aligned carve-up (the swizzled TMA boxes want aligned bases);
  // offsets from smem_raw keep the pointers in the shared window (LDS/STS,
  // not generic loads and stores)
  unsigned char* base = smem_raw + ((1024u - (saddr(smem_raw) & 1023u)) & 1023u);
  unsigned char* astage = base;                                       // kAStages x 16 KB
  unsigned char* dstage = astage + kAStages * kAStageBytes;           // kDStages x 24 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(dstage + kDStages * kDStageBytes);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kAStages;
  uint64_t* d_full = a_empty + kAStages;
  uint64_t* d_empty = d_full + kDStages;
  uint64_t* acc_full = d_empty + kDStages;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* info_full = acc_empty + 1;   // span metadata published by the issuer
  uint64_t* desc_empty = info_full + 1;  // 2: span exponent descriptors free
  uint64_t* meta_full = desc_empty + 2;  // kAStages: the scout's decision for the chunk in A slot s
  uint64_t* half_full = meta_full + kAStages;  // kDStages: this CTA's half of the slot is written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(half_full + kDStages);
  int* d_meta = reinterpret_cast<int*>(tmem_slot + 4);   // kDStages: chunk starts a span
  int* span_last = d_meta + kDStages;                    // issuer -> drain: this span is the last
  int* desc = span_last + 4;                             // [2][128] span exponents
  int* meta = desc + 2 * kCB;                            // [kAStages][2]: fresh, span
  int* sbad = meta + 2 * kAStages;                       // [128]
  int* dsq = sbad + kCB;                                 // [2][128] D8 diagonal sums per span (group 1's MMA warp)
  uint32_t* pmax = reinterpret_cast<uint32_t*>(dsq + 2 * kCB);  // [kPmaxSlots][128] the peer half's column maxima
  uint64_t* pmax_full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(pmax + kPmaxSlots * kCB) + 7) & ~(uintptr_t)7);  // [kPmaxSlots]
  static_assert(kPmaxSlots > kAStages + kDStages + 1, "the peer's maxima ring must outrun both pipelines");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x >> 1, g = blockIdx.x & 1;
  // timing probes (MPSVD_OZ32_DBG, results wrong): bit 0 skips the MMAs,
  // bit 1 the digit conversion (zeros are written), bit 2 the scouts' peer
  // exchange and barrier reductions
  const int kdbg = wmode >> 8;
  wmode &= 0xFF;
  const uint32_t zmask = (uint32_t)kdbg >> 16;  // 0, unknown to the compiler
  OZ32_DBG(const Oz32Dbg dbg = g_oz32_dbg;)
  const long long nch_all = c_end - c_begin;
  const long long c0 = c_begin + nch_all * pair / npairs, c1 = c_begin + nch_all * (pair + 1) / npairs;
  const int nchunk = (int)(c1 - c0);
  const int nch = (nchunk + kStep - 1) / kStep;  // steps; the last may hold one chunk (the other is zero)

  if (threadIdx.x == 0) {
    for (int i = 0; i < kAStages; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], kGroupWarps + kScoutWarps);  // the chunk's converter group + the scouts
      mbar_init(&meta_full[i], kScoutWarps);
    }
    for (int i = 0; i < kDStages; ++i) {
      mbar_init(&d_full[i], kGroupWarps);  // own converter warps (+ the peer's half: transaction bytes)
      mbar_init(&d_empty[i], 2);           // the MMAs of both CTAs have read the slot
      mbar_init(&half_full[i], kGroupWarps);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
    mbar_init(info_full, 1);
    mbar_init(&desc_empty[0], 4);
    mbar_init(&desc_empty[1], 4);
    for (int i = 0; i < kPmaxSlots; ++i) mbar_init(&pmax_full[i], 1);  // one local expect_tx + 512 peer bytes
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < kCB) sbad[threadIdx.x] = 0;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(saddr(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // the peer's barriers are initialised before any remote arrive / store
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&amap) : "memory");
      for (int j = 0; j < nch; ++j) {
        const int s = j % kAStages;
        mbar_wait_m(&a_empty[s], ((unsigned)(j / kAStages) & 1u) ^ 1u, wmode, 64);
        OZ32_DBG(oz32_stamp(dbg, g, pair, j, 0);)
        if (2 * j + g < nchunk) {
          mbar_expect_tx(&a_full[s], kAStageBytes);
          tma_load_2d(astage + (size_t)s * kAStageBytes, &amap, (int)((c0 + 2 * j + g) * kKC), 0, &a_full[s]);
        } else {
          mbar_arrive(&a_full[s]);  // odd tail: this CTA's chunk of the last step is all zero
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: the whole warp runs the loop (warp-uniform control
    // flow keeps the descriptors in uniform registers; a divergent one-lane
    // loop paid ~150 cycles of register traffic per MMA) and lane 0's
    // instructions are the only ones enabled
    const uint32_t lead = lane == 0;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kCB >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);  // D s32, A/B s8 K-major, N = M = 128
    const uint32_t idesc2 = (idesc & ~(63u << 17)) | ((uint32_t)(256 >> 3) << 17);  // the same with N = 256
    const uint64_t dbase = kdesc(saddr(dstage));           // + (byte offset >> 4) per operand
    // D8 diagonal (group 1): sum over the chunk's 32 rows of d_4^2 per
    // column, from digit plane 4 of both halves of the slot; lane l owns
    // columns l + 32 k (each 8-lane group reads 128 contiguous bytes)
    int s8[4] = {0, 0, 0, 0};
    int span = -1;
    for (int j = 0; j < nch; ++j) {
      const int s = j % kDStages;
      mbar_wait_cl(&d_full[s], (unsigned)(j / kDStages) & 1u);
      const bool fresh = d_meta[s] != 0;
      if (fresh && g == 1) {
        if (span >= 0)
#pragma unroll
          for (int k = 0; k < 4; ++k) dsq[(span & 1) * kCB + lane + 32 * k] = s8[k];  // the closing span's D8
#pragma unroll
        for (int k = 0; k < 4; ++k) s8[k] = 0;
      }
      OZ32_DBG(if (lead) oz32_stamp(dbg, g, pair, j, 5);)
      OZ32_DBG(if (dbg.fresh && lead) dbg.fresh[(c0 + 2 * j) * 2 + g] = fresh ? 1 : 0;)
      if (fresh) {
        if (span >= 0) {  // close the previous span: the drain may read it
          if (lead) span_last[span & 1] = 0;
          __syncwarp();
          arrive_lead(info_full, lead);
          commit_lead(acc_full, lead);
        }
        ++span;
        mbar_wait_m(acc_empty, (unsigned)span & 1u, wmode, 128);  // its accumulators are drained
      }
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint64_t sd = dbase + (uint64_t)((uint32_t)s * (kDStageBytes >> 4));
      uint32_t dep = 0;
      const uint64_t sd1 = sd + (uint64_t)((2 * kHalfBytes) >> 4);  // the step's second chunk (K-core groups 2, 3)
      if (g == 0) {
        if (!(kdbg & 1)) {
          issue_chunk<0>(tmem, sd, idesc, idesc2, fresh, lead);
          issue_chunk<0>(tmem, sd1, idesc, idesc2, false, lead);
        }
      } else {
        if (!(kdbg & 1)) {
          issue_chunk<1>(tmem, sd, idesc, idesc2, fresh, lead);
          issue_chunk<1>(tmem, sd1, idesc, idesc2, false, lead);
        }
        const unsigned char* p4 = dstage + (size_t)s * kDStageBytes + 3 * 2048 + (lane >> 3) * 128 + (lane & 7) * 16;
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int h = 0; h < 2 * kStep; ++h) {
            const uint4 w = *reinterpret_cast<const uint4*>(p4 + h * kHalfBytes + k * 512);
            s8[k] = __dp4a((int)w.x, (int)w.x, s8[k]);
            s8[k] = __dp4a((int)w.y, (int)w.y, s8[k]);
            s8[k] = __dp4a((int)w.z, (int)w.z, s8[k]);
            s8[k] = __dp4a((int)w.w, (int)w.w, s8[k]);
          }
        // the slot may be refilled once the commit below lands: every lane's
        // loads must have returned first (see release_a)
        dep = __reduce_or_sync(0xffffffffu, (uint32_t)(s8[0] | s8[1] | s8[2] | s8[3]) & zmask);
      }
      commit_lead_pair_dep(&d_empty[s], lead, dep);  // the slot is free (in both CTAs) once these MMAs have read it
      OZ32_DBG(if (lead) oz32_stamp(dbg, g, pair, j, 6);)
    }
    if (g == 1 && span >= 0)
#pragma unroll
      for (int k = 0; k < 4; ++k) dsq[(span & 1) * kCB + lane + 32 * k] = s8[k];  // the last span's D8
    if (lead) span_last[span >= 0 ? (span & 1) : 0] = span >= 0 ? 1 : 2;  // 2: no chunk, nothing to drain
    __syncwarp();
    arrive_lead(info_full, lead);
    if (span >= 0) commit_lead(acc_full, lead);
  } else if (warp == kWarpCopy) {
    // ---- copier: once this CTA's converters have written their half of
    // digit slot s, one bulk copy moves it into the peer's slot s, completing
    // on the peer's d_full (transaction bytes). Group 1 does not use digit 6,
    // so group 0 sends digits 1-5 only.
    if (lane == 0) {
      const uint32_t peer = (uint32_t)(g ^ 1);
      const uint32_t src0 = saddr(dstage) + (uint32_t)(g * 2 * kHalfBytes);  // this CTA's chunk: K-core groups 2g, 2g+1
      const uint32_t dst0 = mapa(src0, peer);
      const uint32_t bar0 = mapa(saddr(d_full), peer);
      const unsigned bytes = 2u * kHalfBytes;
      for (int j = 0; j < nch; ++j) {
        const int s = j % kDStages;
        mbar_wait_m(&half_full[s], (unsigned)(j / kDStages) & 1u, wmode, 0);
        OZ32_DBG(oz32_stamp(dbg, g, pair, j, 4);)
        bulk_s2peer(dst0 + (uint32_t)(s * kDStageBytes), src0 + (uint32_t)(s * kDStageBytes), bytes,
                    bar0 + (uint32_t)(s * 8));
      }
    }
  } else if (warp >= kScoutWarp0) {
    // ---- scouts: lane owns column c = 32 (warp - kScoutWarp0) + lane; per
    // chunk the column maximum (finite entries), the span decision (first
    // chunk, span_max chunks, or an entry >= 2^E_c: OR over the 128 scout
    // threads) and at a new span E_c = e(max) + kHead
    const int c = (warp - kScoutWarp0) * 32 + lane;
    const uint32_t pmax_peer = mapa(saddr(pmax), (uint32_t)(g ^ 1));
    const uint32_t pmax_full_peer = mapa(saddr(pmax_full), (uint32_t)(g ^ 1));
    int Ec = kZeroE;
    int span = -1, len = 0;
    // the local part of step jj: this CTA's column maxima, the A slot
    // released, the value sent to the peer. It runs one step ahead of the
    // decision, so the exchange's round trip overlaps the next step's scan.
    auto scan = [&](int jj) -> uint32_t {
      const int sa = jj % kAStages;
      if (warp == kScoutWarp0) mbar_wait_m(&a_full[sa], (unsigned)(jj / kAStages) & 1u, wmode, 0);
      nbar_sync(7, 128);
      const unsigned char* colp = astage + (size_t)sa * kAStageBytes + (size_t)c * 128;
      // max of |x| as bit patterns over this CTA's chunk of the step: inf /
      // NaN (exponent 255) lie above every finite value, so they force a new
      // span and a huge E_c for their column, whose entries the converters
      // then zero and flag
      uint32_t m = 0;
      if (2 * jj + g < nchunk)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint4 w = *reinterpret_cast<const uint4*>(colp + ((u ^ (c & 7)) << 4));
          m = max(m, max(max(w.x & 0x7FFFFFFFu, w.y & 0x7FFFFFFFu), max(w.z & 0x7FFFFFFFu, w.w & 0x7FFFFFFFu)));
        }
      release_a(&a_empty[sa], lane, m, zmask);
      // send the half maxima to the peer (st.async, completing on its
      // pmax_full): both CTAs of the pair decide from the same 64 rows. The
      // peer is never more than the A + digit ring depths (+1) ahead
      // (kPmaxSlots exceeds that), so a slot is never overwritten before
      // this CTA has read it.
      if (!(kdbg & 4)) {
        const int ps = jj % kPmaxSlots;
        if (threadIdx.x == kScoutWarp0 * 32) mbar_expect_tx(&pmax_full[ps], kCB * 4);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(
                         pmax_peer + (uint32_t)((ps * kCB + c) * 4)),
                     "r"(m), "r"(pmax_full_peer + (uint32_t)(ps * 8))
                     : "memory");
      }
      return m;
    };
    uint32_t mloc = nch > 0 ? scan(0) : 0u;
    for (int j = 0; j < nch; ++j) {
      const int sa = j % kAStages;
      uint32_t mx = mloc;
      if (j + 1 < nch) mloc = scan(j + 1);
      if (!(kdbg & 4)) {
        const int ps = j % kPmaxSlots;
        mbar_wait_cl(&pmax_full[ps], (unsigned)(j / kPmaxSlots) & 1u);
        mx = max(mx, pmax[ps * kCB + c]);
      }
      // bit 0: some column needs a new span; bit 1: some entry is inf / NaN
      const uint32_t mine = (fexp_bits(mx) > Ec ? 1u : 0u) | (mx >= 0x7F800000u ? 2u : 0u);
      uint32_t any = 0, anybad = 0;
      if (!(kdbg & 4)) {
      asm volatile(
          "{\n.reg .pred p, q;\nsetp.ne.u32 p, %1, 0;\nbar.red.or.pred q, 1, 128, p;\nselp.u32 %0, 1, 0, q;\n}\n"
          : "=r"(any)
          : "r"(mine & 1u)
          : "memory");
      asm volatile(
          "{\n.reg .pred p, q;\nsetp.ne.u32 p, %1, 0;\nbar.red.or.pred q, 1, 128, p;\nselp.u32 %0, 1, 0, q;\n}\n"
          : "=r"(anybad)
          : "r"(mine & 2u)
          : "memory");
      }
      const bool fresh = any != 0 || len == span_max || j == 0;
      if (fresh) {
        ++span;
        len = 0;
        if (span >= 2) mbar_wait_m(&desc_empty[span & 1], ((unsigned)(span >> 1) & 1u) ^ 1u, wmode, 256);
        Ec = mx ? fexp_bits(mx) + kHead : kZeroE;
        desc[(span & 1) * kCB + c] = Ec;
      }
      ++len;
      if (c == 0) {
        meta[2 * sa] = (fresh ? 1 : 0) | (anybad ? 2 : 0);
        meta[2 * sa + 1] = span;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&meta_full[sa]);
      OZ32_DBG(if (threadIdx.x == kScoutWarp0 * 32) oz32_stamp(dbg, g, pair, j, 1);)
    }
  } else if (warp < kConvWarp0) {
    // ---- drain: a warp may only touch TMEM lanes 32 (warp % 4) .. + 31, so
    // lane quarter qd = warp % 4; thread = tile row i
    const int qd = warp & 3;
    const int i = qd * 32 + lane;
    if (lane == 0) mbar_arrive(acc_empty);  // the accumulators start free
    double2* P = partials + (size_t)blockIdx.x * kCB * kCB;
    for (int span = 0;; ++span) {
      if (warp == 2) mbar_wait_m(info_full, (unsigned)span & 1u, wmode, 0);
      nbar_sync(6, 128);
      const int last = span_last[span & 1];
      if (last == 2) {  // empty range: the partial is zero
        if (!accumulate && i < n)
          for (int jj = 0; jj < n; ++jj) P[(size_t)jj * kCB + i] = make_double2(0.0, 0.0);
        break;
      }
      mbar_wait_m(acc_full, (unsigned)span & 1u, wmode, 256);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int* E = desc + (span & 1) * kCB;
      const int ei = E[i];
      const int basee = g ? 47 : 40;
      // 4 columns per step (4 x 4 TMEM words, 4 running partials in flight):
      // the kernel runs 27 warps, so the drain must fit in ~72 registers
      // the partials of column group j0 + 4 are requested before group j0 is
      // combined, so their L2 / HBM round trip overlaps the dd arithmetic
      const bool rmw = accumulate || span > 0;
      double2 nxt[4];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
        nxt[jj] = (rmw && i < n && jj < n) ? P[(size_t)jj * kCB + i] : make_double2(0.0, 0.0);
      for (int j0 = 0; j0 < kCB; j0 += 4) {
        uint32_t v[4][4];
        const uint32_t taddr = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)j0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                       : "=r"(v[k][0]), "=r"(v[k][1]), "=r"(v[k][2]), "=r"(v[k][3])
                       : "r"(taddr + (uint32_t)(k * kCB)));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (i < n) {
          // the running partials of the step are loaded together (one
          // memory latency per group of columns, not per entry)
          double2 old[4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            old[jj] = nxt[jj];
            nxt[jj] = (rmw && j0 + 4 + jj < n) ? P[(size_t)(j0 + 4 + jj) * kCB + i] : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int jc = j0 + jj;
            if (jc >= n) continue;
            // accumulator columns: group 0 {T7, T3, T4, D2}, group 1 {T5, T6, D4, D6} (issue_chunk)
            dd t0 = g == 0 ? group_total(0, (int)v[0][jj], (int)v[2][jj], (int)v[1][jj], (int)v[3][jj])
                           : group_total(1, (int)v[1][jj], (int)v[0][jj], (int)v[2][jj], (int)v[3][jj]);
            if (g == 1 && jc == i)  // D8 diagonal: sum d_4^2 at 2^-16 of this frame (halved)
              t0 = dd_add(t0, dd_make((double)dsq[(span & 1) * kCB + i] * 0x1p-16, 0.0));
            const int sc = ei + E[jc] - 92 + basee;
            dd t = dd_make(scalbn(t0.hi, sc), scalbn(t0.lo, sc));
            if (rmw) t = dd_add(dd_make(old[jj].x, old[jj].y), t);
            P[(size_t)jc * kCB + i] = make_double2(t.hi, t.lo);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(acc_empty);
        mbar_arrive(&desc_empty[span & 1]);
      }
      if (last) break;
    }
  } else {
    // ---- converters: thread = (column c, rows 16 q .. 16 q + 15 of this
    // CTA's chunk of the step). Each CTA converts its own chunk (K-core
    // groups 2g, 2g+1 of the step's digit slot); the copier moves it into the
    // peer's slot (one bulk copy through distributed shared memory), so the
    // pair converts each row once. A slot is full when this CTA's converter
    // warps have arrived and the peer's chunk has landed (transaction
    // bytes), and free when both CTAs' MMAs have read it (multicast commit).
    // Two groups of 8 warps alternate steps (group G takes j = G mod 2), so
    // the per-step hand-off latencies of one group overlap the other's work.
    const int grp = (threadIdx.x - kConvWarp0 * 32) >> 8;
    const int t = (threadIdx.x - kConvWarp0 * 32) & 255;
    // warp w of the group: K-core group q = w & 1, columns 32 (w >> 1) ..
    // + 31, so a warp's 16-byte digit stores are 512 contiguous bytes and its
    // A loads hit 8 distinct 16-byte units per 8 lanes (no bank conflicts)
    const int q = (t >> 5) & 1, c = (t & 31) + 32 * (t >> 6);
    const int gw = t >> 5;            // warp within the group
    const uint32_t dloc = saddr(dstage) + (uint32_t)((2 * g + q) * kHalfBytes + (c >> 3) * 128 + (c & 7) * 16);
    const unsigned in_bytes = 2u * kHalfBytes;  // the peer's chunk
    int E = kZeroE;
    int span = -1;
    int badc = 0;
    for (int j = grp; j < nch; j += kConvGroups) {
      const int sa = j % kAStages;
      const bool valid = 2 * j + g < nchunk;
      OZ32_DBG(if (t == 0) oz32_stamp(dbg, g, pair, j, 8);)  // iteration start
      // one warp of the group polls; the group's other warps block on a
      // named barrier (polling by all 16 converter warps took most of the
      // SM's issue slots, ncu)
      if (gw == 0) {
        mbar_wait_m(&meta_full[sa], (unsigned)(j / kAStages) & 1u, wmode, 0);
        mbar_wait_m(&a_full[sa], (unsigned)(j / kAStages) & 1u, wmode, 0);
      }
      OZ32_DBG(if (t == 0) oz32_stamp(dbg, g, pair, j, 9);)
      nbar_sync(2 + 2 * grp, 256);
      OZ32_DBG(if (t == 0) oz32_stamp(dbg, g, pair, j, 10);)
      const int mflags = meta[2 * sa];
      const bool fresh = (mflags & 1) != 0;
      const int mspan = meta[2 * sa + 1];
      // 16 values: 16-byte units 4 q .. 4 q + 3 of column c's 128 B, 128B-swizzled
      const unsigned char* col = astage + (size_t)sa * kAStageBytes + (size_t)c * 128;
      uint32_t b[16];
      if (valid) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint4 w = *reinterpret_cast<const uint4*>(col + (((4 * q + u) ^ (c & 7)) << 4));
          b[4 * u] = w.x;
          b[4 * u + 1] = w.y;
          b[4 * u + 2] = w.z;
          b[4 * u + 3] = w.w;
        }
      } else {
#pragma unroll
        for (int r = 0; r < 16; ++r) b[r] = 0;  // odd tail: the chunk beyond the range is zero
      }
      release_a(&a_empty[sa], lane, b[0] | b[4] | b[8] | b[12] | (uint32_t)mflags, zmask);
      OZ32_DBG(if (t == 0) oz32_stamp(dbg, g, pair, j, 11);)
      if (mflags & 2) {  // inf / NaN in this step (the scouts saw it): flag the column, use zeros
#pragma unroll
        for (int r = 0; r < 16; ++r)
          if ((b[r] & 0x7FFFFFFFu) >= 0x7F800000u) {
            b[r] = 0;
            badc = 1;
          }
      }
      if (mspan != span) {  // this group's first step of a span (it may have skipped a short one)
        span = mspan;
        E = desc[(span & 1) * kCB + c];
      }
      const int sd = j % kDStages;
      OZ32_DBG(if (t == 0) oz32_stamp(dbg, g, pair, j, 7);)  // A data in registers
      if (gw == 0) mbar_wait_m(&d_empty[sd], ((unsigned)(j / kDStages) & 1u) ^ 1u, wmode, 0);
      nbar_sync(3 + 2 * grp, 256);
      OZ32_DBG(if (t == 0) oz32_stamp(dbg, g, pair, j, 2);)
      if (t == 0) d_meta[sd] = fresh ? 1 : 0;
      uint32_t ylo[16], yhi[16];
      if (kdbg & 2) {
#pragma unroll
        for (int r = 0; r < 16; ++r) ylo[r] = yhi[r] = 0x80808080u;
      } else if (__all_sync(0xffffffffu, E >= -78 || E == kZeroE)) {
        const uint32_t kc = (uint32_t)(942 - (E == kZeroE ? 0 : E)) << 20;
#pragma unroll
        for (int r = 0; r < 16; ++r) fixed48_fast(b[r], kc, ylo[r], yhi[r]);
      } else {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const unsigned long long y = fixed48(b[r], E);
          ylo[r] = (uint32_t)y;
          yhi[r] = (uint32_t)(y >> 32);
        }
      }
      // 4 x 4 byte transposes: plane word w of digit p = byte (6 - p) of Y
      // for rows 4w .. 4w + 3 (8 PRMT for the low word's 4 digits, 4 for the
      // high word's 2, per 4 rows); then XOR 0x80 per byte (balanced digits)
      uint32_t o[6][4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t a01 = __byte_perm(ylo[4 * w], ylo[4 * w + 1], 0x5140);
        const uint32_t b01 = __byte_perm(ylo[4 * w], ylo[4 * w + 1], 0x7362);
        const uint32_t a23 = __byte_perm(ylo[4 * w + 2], ylo[4 * w + 3], 0x5140);
        const uint32_t b23 = __byte_perm(ylo[4 * w + 2], ylo[4 * w + 3], 0x7362);
        const uint32_t c01 = __byte_perm(yhi[4 * w], yhi[4 * w + 1], 0x5140);
        const uint32_t c23 = __byte_perm(yhi[4 * w + 2], yhi[4 * w + 3], 0x5140);
        o[5][w] = __byte_perm(a01, a23, 0x5410) ^ 0x80808080u;  // byte 0: digit 6
        o[4][w] = __byte_perm(a01, a23, 0x7632) ^ 0x80808080u;  // byte 1: digit 5
        o[3][w] = __byte_perm(b01, b23, 0x5410) ^ 0x80808080u;  // byte 2: digit 4
        o[2][w] = __byte_perm(b01, b23, 0x7632) ^ 0x80808080u;  // byte 3: digit 3
        o[1][w] = __byte_perm(c01, c23, 0x5410) ^ 0x80808080u;  // byte 4: digit 2
        o[0][w] = __byte_perm(c01, c23, 0x7632) ^ 0x80808080u;  // byte 5: digit 1
      }
      const uint32_t so = dloc + (uint32_t)(sd * kDStageBytes);
#pragma unroll
      for (int p = 1; p <= kDigits; ++p)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(so + (uint32_t)((p - 1) * 2048)),
                     "r"(o[p - 1][0]), "r"(o[p - 1][1]), "r"(o[p - 1][2]), "r"(o[p - 1][3])
                     : "memory");
      OZ32_DBG(if (dbg.digits && valid) {
        const long long gc = c0 + 2 * j + g;
        for (int p = 1; p <= kDigits; ++p)
          *reinterpret_cast<uint4*>(dbg.digits + ((gc * kDigits + p - 1) * kCB + c) * 32 + 16 * q) =
              make_uint4(o[p - 1][0], o[p - 1][1], o[p - 1][2], o[p - 1][3]);
        if (q == 0) dbg.E[gc * kCB + c] = (short)E;
      })
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> tensor core / bulk copy
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&half_full[sd]);
        OZ32_DBG(if (t == 0) oz32_stamp(dbg, g, pair, j, 3);)
        if (t == 0)
          mbar_expect_tx(&d_full[sd], in_bytes);  // one of the arrivals also expects the peer's chunk
        else
          mbar_arrive(&d_full[sd]);
      }
    }
    // the peer's MMAs arrive (multicast) on this CTA's slot barriers: wait
    // for the last arrivals before this CTA may exit
    if (grp == 0)
      for (int jj = nch; jj < nch + kDStages; ++jj)
        if (jj >= kDStages) mbar_wait_m(&d_empty[jj % kDStages], ((unsigned)(jj / kDStages) & 1u) ^ 1u, wmode, 32);
    if (badc) atomicOr(&sbad[c], 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  cluster_sync_all();  // no remote store or arrive targets this CTA after it exits
  if (threadIdx.x < kCB && threadIdx.x < n && sbad[threadIdx.x]) atomicOr(&bad_cols[threadIdx.x], 1);
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

// M (n x n, both triangles) = fl64(sum over CTAs of P(i,j) + P(j,i)), in CTA order
__global__ void __launch_bounds__(256)
gram_f32_ozaki_combine(const double2* __restrict__ partials, int ncta, int n, const int* __restrict__ bad_cols,
                       double* __restrict__ m_out) {
  const int nn = n * n;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += gridDim.x * blockDim.x) {
    const int j = e / n, i = e - j * n;
    if (i > j) continue;
    dd acc = dd_make(0.0, 0.0);
    for (int k = 0; k < ncta; ++k) {
      const double2* P = partials + (size_t)k * kCB * kCB;
      const double2 a = P[(size_t)j * kCB + i], b = P[(size_t)i * kCB + j];
      acc = dd_add(acc, dd_make(a.x, a.y));
      acc = dd_add(acc, dd_make(b.x, b.y));
    }
    double v = acc.hi;
    if (bad_cols[i] || bad_cols[j]) v = __longlong_as_double(0x7ff8000000000000ll);
    m_out[(size_t)j * n + i] = v;
    m_out[(size_t)i * n + j] = v;
  }
}

// ---------------------------------------------------------------------------
static size_t ozaki32_smem(int astages, int dstages) {
  return 1024 + (size_t)astages * kAStageBytes + (size_t)dstages * kDStageBytes + 1024 + 4 * kCB * 4 + kCB * 4 +
         4 * kCB * 4 + 64 * 4 + (size_t)kPmaxSlots * kCB * 4 + kPmaxSlots * 8;
}

// pipeline shape (MPSVD_OZ32_STAGES: "4x3" (default), "3x3", "6x2", "5x2": A x digit slots) and
// wait mode (MPSVD_OZ32_WAIT: 0 hinted try_wait, 1 plain try_wait, 2
// back-off), read once
struct Oz32Cfg {
  int astages = 4, dstages = 3;  // A slots (16 KB) x digit slots (48 KB, a 64-row step)
  int wmode = 2;
};
static const Oz32Cfg& oz32_cfg() {
  static Oz32Cfg c;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* st = getenv("MPSVD_OZ32_STAGES");
    if (st && st[0] >= '3' && st[0] <= '9' && st[1] == 'x' && st[2] >= '2' && st[2] <= '9') {
      c.astages = st[0] - '0';
      c.dstages = st[2] - '0';
    }
    const char* w = getenv("MPSVD_OZ32_WAIT");
    if (w && w[0] >= '0' && w[0] <= '2') c.wmode = w[0] - '0';
    const char* d = getenv("MPSVD_OZ32_DBG");
    if (d) c.wmode |= (atoi(d) & 7) << 8;
  });
  return c;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    else
      cudaGetLastError();
  });
  return fn;
}

bool gram_ozaki32_supported(const float* a, long long lda, long long m, int n) {
  return n >= 1 && n <= kCB && m >= 1 && (reinterpret_cast<uintptr_t>(a) % 16 == 0) && (lda % 4 == 0) &&
         lda < (1LL << 38) && encode_fn() != nullptr;
}

// CTA pairs (clusters of 2) that can be resident at once: the launch must
// fit one wave (a second wave of a few pairs would double the range's time)
using Oz32Kern = void (*)(CUtensorMap, int, long long, long long, int, double2*, int*, int, int, int);
static Oz32Kern oz32_kernel(const Oz32Cfg& c) {
  const int k = c.astages * 10 + c.dstages;
  switch (k) {
    case 33: return gram_f32_ozaki<3, 3>;
    case 62: return gram_f32_ozaki<6, 2>;
    case 52: return gram_f32_ozaki<5, 2>;
    default: return gram_f32_ozaki<4, 3>;
  }
}

int gram_ozaki32_max_pairs() {
  const Oz32Cfg& cfg = oz32_cfg();
  auto kern = oz32_kernel(cfg);
  const size_t smem = ozaki32_smem(cfg.astages, cfg.dstages);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(2);
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, kern, &lc) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return nc;
}

size_t gram_ozaki32_partial_bytes(int npairs) { return (size_t)2 * npairs * kCB * kCB * sizeof(double2); }

cudaError_t launch_gram_ozaki32_begin(int* bad_cols, cudaStream_t st) {
  return cudaMemsetAsync(bad_cols, 0, kCB * sizeof(int), st);
}

cudaError_t launch_gram_ozaki32_range(const float* a, long long lda, long long m, int n, long long c_begin,
                                      long long c_end, int npairs, double2* partials, int* bad_cols, bool accumulate,
                                      cudaStream_t st) {
  auto enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)lda * 4};
  const cuuint32_t box[2] = {(cuuint32_t)kKC, (cuuint32_t)kCB};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const Oz32Cfg& cfg = oz32_cfg();
  auto kern = oz32_kernel(cfg);
  const size_t smem = ozaki32_smem(cfg.astages, cfg.dstages);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // test hook: steps (64 rows) per exact span (MPSVD_OZAKI32_SPAN, at most kSpanMax)
  const char* span_env = getenv("MPSVD_OZAKI32_SPAN");
  int span_max = span_env && atoi(span_env) > 0 ? atoi(span_env) : kSpanMax;
  if (span_max > kSpanMax) span_max = kSpanMax;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(2 * npairs);
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;  // CTA pair = cluster of 2 (distributed shared memory)
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, kern, map, n, c_begin, c_end, npairs, partials, bad_cols, accumulate ? 1 : 0,
                            span_max, cfg.wmode);
}

cudaError_t launch_gram_ozaki32_combine(const double2* partials, int npairs, int n, const int* bad_cols,
                                        double* m_out, cudaStream_t st) {
  const int nn = n * n;
  int grid = (nn + 255) / 256;
  if (grid > 148 * 4) grid = 148 * 4;
  gram_f32_ozaki_combine<<<grid, 256, 0, st>>>(partials, 2 * npairs, n, bad_cols, m_out);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace mpsvd
