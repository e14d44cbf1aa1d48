// K4 / K5: two-sided Jacobi eigensolver on the n x n Gram matrix, fp64 (K4)
// or double-double (K5), plus the V replay and the sort/sign/sigma epilogue.
//
// Reference semantics: twosided_impl (proj/src/jacobi.cpp:189-264):
//   * skip a pair when |a_ij| <= tol * sqrt(a_ii) * sqrt(a_jj) (the product of
//     square roots, jacobi.cpp:211-217), tol = n*u (jacobi.cpp:274-275);
//   * zeta = (a_jj - a_ii) / (2 a_ij), t = sign(zeta)/(|zeta| + hypot(1, zeta)),
//     c = 1/hypot(1, t), s = c t (jacobi.cpp:219-224);
//   * a_ii -= t a_ij, a_jj += t a_ij, a_ij = 0 exactly, PD re-check
//     (jacobi.cpp:236-243); converged after a sweep without rotations,
//     NoConvergenceError after max_sweeps (jacobi.cpp:256-262);
//   * stable descending sort, V's first largest entry made >= 0
//     (jacobi.cpp:280-304).
//
// Device schedule: parallel round-robin. A sweep is N-1
// rounds of N/2 disjoint pairs (N = n rounded up to even). Every CTA computes
// all rotations of the round redundantly from a small double-buffered
// "next diagonal blocks" array, so the whole grid agrees on convergence and
// positive-definiteness without extra communication, and a round needs ONE
// grid-wide barrier: the threads then update all 2x2 blocks between pairs
// (column rotation of the higher pair first, then the row rotation of the
// lower pair), each element owned by exactly one thread, and publish the
// entries the next round's rotations will read. Small matrices (n^2 entries
// fit in shared memory) run in a single CTA with A resident in smem.
// Rotations are logged (c, s) and V is rebuilt afterwards by an
// embarrassingly parallel replay over its rows (rows of V never mix).
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace mpsvd {
namespace dev {

// ---------------------------------------------------------------------------
// Arithmetic traits: ST = storage type, AT = arithmetic type.
template <typename ST>
struct Arith;

template <>
struct Arith<double> {
  using AT = double;
  static __device__ __forceinline__ AT ldg(const double* p) { return __ldcg(p); }
  static __device__ __forceinline__ AT lds(const double* p) { return *p; }
  static __device__ __forceinline__ void st(double* p, AT v) { *p = v; }
  static __device__ __forceinline__ AT zero() { return 0.0; }
  static __device__ __forceinline__ AT one() { return 1.0; }
  static __device__ __forceinline__ double hi(AT v) { return v; }
  static __device__ __forceinline__ bool gt0(AT v) { return v > 0.0; }
  static __device__ __forceinline__ bool is_identity(AT c, AT s) { return s == 0.0 && c == 1.0; }
  static __device__ __forceinline__ AT rot_lo(AT c, AT s, AT x, AT y) { return fma(c, x, -(s * y)); }
  static __device__ __forceinline__ AT rot_hi(AT c, AT s, AT x, AT y) { return fma(s, x, c * y); }
  // Stop test of jacobi.cpp:211-217, |a_pq| <= tol sqrt(a_pp) sqrt(a_qq), with
  // one square root of the product; the two-root form only when the product
  // leaves the normal range (the reference's reason for it).
  static __device__ __forceinline__ bool active(AT app, AT aqq, AT apq, double tol) {
    const double pr = app * aqq;
    const double thresh = (pr > 0x1p-1000 && pr < 0x1p1000) ? tol * sqrt(pr) : tol * sqrt(app) * sqrt(aqq);
    return !(fabs(apq) <= thresh);
  }
  // normalised off-diagonal |a_pq| / sqrt(a_pp a_qq) (NoConvergence payload)
  static __device__ __forceinline__ double ratio(AT app, AT aqq, AT apq) { return fabs(apq) / sqrt(app * aqq); }
  // Annihilating rotation (jacobi.cpp:219-241). With x = a_qq - a_pp,
  // y = 2 a_pq, q = x^2 + y^2, r = sqrt(q):
  //   t = sign(x) y / (|x| + r)        (= sign(zeta)/(|zeta| + hypot(1, zeta))),
  //   c = sqrt(1/2 + 1/2 |x| / r)      (= 1/sqrt(1 + t^2)),   s = c t,
  // t = +1 at x == 0 (the reference's sign(0) = +1). 1/r is formed as
  // r (1/q) with the division next to the square root (both need only q), so
  // the dependent chain holds two long operations (sqrt|div, then div|sqrt)
  // instead of the reference's five; x and y are scaled by an exact power of
  // two when q would leave the normal range (t, c, s are scale-free).
  // Diagonal: a_pp - t a_pq, a_qq + t a_pq (fused).
  static __device__ __forceinline__ void rotate(AT app, AT aqq, AT apq, AT& c, AT& s, AT& npp, AT& nqq) {
    double x = aqq - app, y = 2.0 * apq;
    const bool xzero = x == 0.0, xpos = x > 0.0;  // before any rescaling (it may flush a tiny x)
    const double big = fmax(fabs(x), fabs(y));
    if (!(big < 0x1p500 && big > 0x1p-500)) {
      const double2 xy = rescale(x, y, big);
      x = xy.x;
      y = xy.y;
    }
    const double ax = fabs(x);
    const double q = fma(x, x, y * y);
    const double ys = xpos ? y : -y;
    double t;
    // operands and results far inside the normal range: the branch-free
    // forms of sqrt and / (common.cuh, the same bits), whose independent
    // pairs (sqrt q | 1 / q, then y / den | sqrt c^2) overlap
    if (big < 0x1p400 && big > 0x1p-400 && fabs(y) > big * 0x1p-200) {
      const double r = fast_sqrt_normal(q), iq = fast_div_normal(1.0, q);
      const double den = ax + r;
      t = xzero ? 1.0 : fast_div_normal(ys, den);
      c = fast_sqrt_normal(fma(0.5, ax * (r * iq), 0.5));
    } else {
      const double r = sqrt(q), iq = 1.0 / q;
      const double den = ax + r;
      t = xzero ? 1.0 : ys / den;
      c = sqrt(fma(0.5, ax * (r * iq), 0.5));
    }
    s = c * t;
    npp = fma(-t, apq, app);
    nqq = fma(t, apq, aqq);
  }
  static __device__ __noinline__ double2 rescale(double x, double y, double big) {
    int e;  // exact power-of-two rescaling keeps x^2 + y^2 finite and normal
    frexp(big, &e);
    return make_double2(ldexp(x, -e), ldexp(y, -e));
  }
};

template <>
struct Arith<double2> {
  using AT = dd;
  static __device__ __forceinline__ AT ldg(const double2* p) {
    const double2 v = __ldcg(p);
    return dd_make(v.x, v.y);
  }
  static __device__ __forceinline__ AT lds(const double2* p) {
    const double2 v = *p;
    return dd_make(v.x, v.y);
  }
  static __device__ __forceinline__ void st(double2* p, AT v) { *p = make_double2(v.hi, v.lo); }
  static __device__ __forceinline__ AT zero() { return dd_from(0.0); }
  static __device__ __forceinline__ AT one() { return dd_from(1.0); }
  static __device__ __forceinline__ double hi(AT v) { return v.hi; }
  static __device__ __forceinline__ bool gt0(AT v) { return dd_gt0(v); }
  static __device__ __forceinline__ bool is_identity(AT c, AT s) {
    return s.hi == 0.0 && s.lo == 0.0 && c.hi == 1.0 && c.lo == 0.0;
  }
  static __device__ __forceinline__ AT rot_lo(AT c, AT s, AT x, AT y) {
    return dd_sub(dd_mul(c, x), dd_mul(s, y));
  }
  static __device__ __forceinline__ AT rot_hi(AT c, AT s, AT x, AT y) {
    return dd_add(dd_mul(s, x), dd_mul(c, y));
  }
  // The stop test of the double-double solver is evaluated on the leading
  // words (a relative 2^-53 wobble of a 2^-104-scale threshold is immaterial).
  static __device__ __forceinline__ bool active(AT app, AT aqq, AT apq, double tol) {
    const double pr = app.hi * aqq.hi;
    const double thresh = (pr > 0x1p-1000 && pr < 0x1p1000) ? tol * sqrt(pr) : tol * sqrt(app.hi) * sqrt(aqq.hi);
    return !(fabs(apq.hi) <= thresh);
  }
  static __device__ __forceinline__ double ratio(AT app, AT aqq, AT apq) {
    return fabs(apq.hi) / sqrt(app.hi * aqq.hi);
  }
  static __device__ __noinline__ double4 rescale(dd x, dd y, double big) {
    int e;
    frexp(big, &e);
    return make_double4(ldexp(x.hi, -e), ldexp(x.lo, -e), ldexp(y.hi, -e), ldexp(y.lo, -e));
  }
  // The rotation of Arith<double>::rotate in double-double. Every quotient
  // and root is one binary64 estimate plus one double-double residual
  // correction (Newton), and each reciprocal is taken next to the square
  // root it belongs to (1/sqrt(v) = sqrt(v) (1/v)), so the dependent chain
  // holds two long operations; dd_sqrt / dd_div (two and three dependent
  // divisions each) made it seven: 5.7 k cycles per rotation at n = 1024.
  //   r = sqrt(q):      r0 = sqrt(q.hi), r = r0 + (q - r0^2) (ir / 2), ir = r0 / q.hi
  //   u = |x| / r:      u0 = |x|.hi ir,  u = u0 + (|x| - u0 r) ir
  //   c = sqrt(c2), c2 = (1 + u) / 2:    c0 = sqrt(c2.hi), c = c0 + (c2 - c0^2) (c0 / c2.hi) / 2
  //   t = +-y / den, den = |x| + r:      id = 1 / (|x|.hi + r0), t0 = y.hi id, t = t0 + (y - t0 den) id
  // Each result carries a relative error of a few 2^-102.
  static __device__ __forceinline__ void rotate(AT app, AT aqq, AT apq, AT& c, AT& s, AT& npp, AT& nqq) {
    dd x = dd_sub(aqq, app), y = dd_scale2(apq);
    const bool xzero = x.hi == 0.0, xpos = x.hi > 0.0;  // before any rescaling
    const double big = fmax(fabs(x.hi), fabs(y.hi));
    if (!(big < 0x1p250 && big > 0x1p-250)) {
      const double4 xy = rescale(x, y, big);
      x = dd_make(xy.x, xy.y);
      y = dd_make(xy.z, xy.w);
    }
    const dd ax = dd_abs(x);
    const dd q = dd_add(dd_mul(x, x), dd_mul(y, y));
    const bool fast = big < 0x1p250 && big > 0x1p-250;  // branch-free sqrt and / (common.cuh, the same bits)
    const double r0 = fast ? fast_sqrt_normal(q.hi) : sqrt(q.hi);
    const double iq = fast ? fast_div_normal(1.0, q.hi) : 1.0 / q.hi;
    const double ir = r0 * iq;
    const double id = fast ? fast_div_normal(1.0, ax.hi + r0) : 1.0 / (ax.hi + r0);
    const dd er = dd_sub(q, two_prod(r0, r0));
    const dd r = quick_two_sum(r0, er.hi * (0.5 * ir));
    const dd den = dd_add(ax, r);
    dd t = dd_from(1.0);
    if (!xzero) {
      const dd ys = xpos ? y : dd_neg(y);
      const double t0 = ys.hi * id;
      const dd et = dd_sub(ys, dd_mul(dd_from(t0), den));
      t = quick_two_sum(t0, et.hi * id);
    }
    const double u0 = ax.hi * ir;
    const dd eu = dd_sub(ax, dd_mul(dd_from(u0), r));
    const dd u = quick_two_sum(u0, eu.hi * ir);
    const dd c2 = dd_add(dd_from(0.5), dd_make(0.5 * u.hi, 0.5 * u.lo));
    const double c0 = fast ? fast_sqrt_normal(c2.hi) : sqrt(c2.hi);
    const double ic2 = fast ? fast_div_normal(1.0, c2.hi) : 1.0 / c2.hi;
    const dd ec = dd_sub(c2, two_prod(c0, c0));
    c = quick_two_sum(c0, ec.hi * (0.5 * (c0 * ic2)));
    s = dd_mul(c, t);
    const dd tapq = dd_mul(t, apq);
    npp = dd_sub(app, tapq);
    nqq = dd_add(aqq, tapq);
  }
};

// ---------------------------------------------------------------------------
constexpr int kJacobiThreads = 256;
// multi-CTA solver: one 512-thread CTA per SM. Every CTA evaluates all of a
// round's rotations (instruction-bound in double-double), so one CTA per SM
// does that work once per SM instead of twice.
constexpr int kJacobiGridThreads = 512;

template <typename ST>
__host__ __device__ constexpr size_t rot_smem_bytes(int np) {
  // c, s, new a_pp, new a_qq (AT each) + packed pair/active word + (multi-CTA)
  // next-round slot and partner of every player (2 x N ints, N = 2 np)
  return (size_t)np * (4 * sizeof(typename Arith<ST>::AT) + sizeof(int)) + (size_t)4 * np * sizeof(int);
}

// Reduction helpers over one warp (all 32 lanes participate).
__device__ __forceinline__ int warp_sum(int v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_min(int v) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// stores into another CTA's shared memory (shared::cluster address from mapa)
__device__ __forceinline__ void st_cluster(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, dd v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(v.hi), "d"(v.lo) : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}

// Optional per-round timestamps of the first sweep (MPSVD_JACOBI_TRACE=1).
__device__ unsigned long long* g_jtrace = nullptr;

template <typename ST, bool kSmem>
__global__ void __launch_bounds__(kSmem ? kJacobiThreads : kJacobiGridThreads)
jacobi_kernel(ST* __restrict__ a_glob, ST* __restrict__ diagbuf, ST* __restrict__ rot_log, int n,
              double tol, int max_sweeps, DevStatus* __restrict__ status, ST* __restrict__ v_out = nullptr,
              int vrows = 0, int vsplit = 0) {
  using A_ = Arith<ST>;
  using AT = typename A_::AT;
  extern __shared__ __align__(16) unsigned char jsm[];
  const int N = n + (n & 1), np = N / 2, R = N - 1;
  const int tid = threadIdx.x, bs = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const long long nblk = (long long)np * (np + 1) / 2;
  const int lda = kSmem ? n + 1 : n;  // odd smem pitch: row and column walks hit distinct banks
  const unsigned FULL = 0xffffffffu;

  // shared memory: [A (smem variant)] [c][s][npp][nqq] [pair word] [block table (smem variant)]
  unsigned char* p = jsm;
  ST* a = a_glob;
  if (kSmem) {
    a = reinterpret_cast<ST*>(p);
    p += (size_t)n * (n + 1) * sizeof(ST);
  }
  AT* rc = reinterpret_cast<AT*>(p);
  AT* rsn = rc + np;
  AT* rnpp = rsn + np;
  AT* rnqq = rnpp + np;
  int* pw = reinterpret_cast<int*>(rnqq + np);  // p | q << 15 | active << 30
  int* blk = pw + np;                            // aa | bb << 16 (smem variant)
  int* nsl = pw + np;                            // multi-CTA: next-round slot | (player is q) << 16
  int* npart = nsl + 2 * np;                     // multi-CTA: next-round partner (n for the bye)
  // fused V (multi-CTA, vrows > 0): this CTA's rows [v0, v0 + vrows) of V,
  // rotated by every round right after the round's rotations are known
  // (rows of V never mix; the separate replay streamed the whole rotation
  // log through every CTA: 259 ms of the c5 eigen phase)
  // (an offset from jsm, not a pointer rebuilt from an integer: the compiler
  // then keeps the shared address space and emits LDS / STS - the rebuilt
  // pointer made every access of the V update a generic LD.E / ST.E)
  const size_t voff = ((size_t)(reinterpret_cast<unsigned char*>(npart + 2 * np) - jsm) + 15) & ~(size_t)15;
  ST* vsm = reinterpret_cast<ST*>(jsm + voff);
  const int v0 = blockIdx.x * vrows, vn = vrows > 0 ? max(0, min(vrows, n - v0)) : 0;
  const int vstep_r = bs / np, vstep_k = bs - vstep_r * np;  // bs = vstep_r * np + vstep_k
  __shared__ int s_flag;
  __shared__ int w_cnt[32], w_bad[32];
  __shared__ double w_worst[32];
  __shared__ unsigned s_sweep_flag;
  // Multi-CTA variant launched as clusters of cs CTAs (n = 1024 dd: the 512
  // double-double rotations of a round are ~6 k cycles of fp64 issue per SM
  // when every CTA evaluates all of them): CTA rank cr evaluates the slots
  // [cr * rchunk, (cr + 1) * rchunk) and stores the results into the shared
  // memory of every CTA of its cluster (distributed shared memory), so each
  // CTA still holds the whole round - same values, same decisions - after
  // one cluster barrier. cs = 1 without a cluster launch.
  constexpr int kMaxCs = 4;
  int cs = 1, cr = 0;
  if (!kSmem) {
    asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(cs));
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(cr));
  }
  const int rchunk = cs > 1 ? ((np + cs - 1) / cs + 31) / 32 * 32 : np;
  const int nw_rot = min(bs, (rchunk + 31) / 32 * 32) / 32;  // warps that own rotation slots
  // shared::cluster address offsets from this CTA's shared memory to the same
  // location in the other CTAs of the cluster (mapa; one offset serves every
  // array). The remote stores are explicit st.shared::cluster: a generic
  // pointer built from a __shared__ one by adding an offset is still treated
  // as CTA-local shared memory by the compiler.
  uint32_t peer_off[kMaxCs - 1] = {0, 0, 0};
  if (!kSmem && cs > 1) {
    const uint32_t self = (uint32_t)__cvta_generic_to_shared(rc);
#pragma unroll
    for (int t = 1; t < kMaxCs; ++t)
      if (t < cs) {
        uint32_t rem;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rem) : "r"(self), "r"((uint32_t)((cr + t) % cs)));
        peer_off[t - 1] = rem - self;
      }
  }
  auto peer = [&](const void* q, int t) { return (uint32_t)__cvta_generic_to_shared(q) + peer_off[t]; };
  // CTA barrier, cluster-wide when the round's rotations are shared
  auto csync = [&]() {
    __syncthreads();  // also reconverges every warp: the cluster barrier below is .aligned
    if (!kSmem && cs > 1)
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  };

  // Grid barrier of the multi-CTA variant (every CTA is resident: the launch
  // is cooperative): a monotonic arrival counter behind the sweep flags,
  // zeroed per launch. Split into arrive / wait so that CTA-local work can
  // sit between the two; the wait ends in csync(). (cg::this_grid().sync()
  // cost ~2.9 k cycles per round at 148 CTAs and is not valid under a
  // cluster launch.)
  unsigned* const gbar = reinterpret_cast<unsigned*>(diagbuf + 6 * np) + 2;
  unsigned gseq = 0;
  auto garrive = [&]() {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(gbar, 1u);
    }
    ++gseq;
  };
  auto gwait = [&]() {
    if (tid == 0) {
      const unsigned target = gseq * gridDim.x;
      unsigned seen;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(seen) : "l"(gbar) : "memory");
      } while ((int)(seen - target) < 0);
    }
    csync();
  };
  auto gsync = [&]() {
    if (kSmem) {
      __syncthreads();
    } else {
      garrive();
      gwait();
    }
  };
  auto LD = [&](const ST* q) -> AT { return kSmem ? A_::lds(q) : A_::ldg(q); };
  auto AE = [&](int row, int col) -> ST* { return a + (long long)col * lda + row; };

  if (kSmem) {
    for (long long e = tid; e < (long long)n * n; e += bs) a[(e / n) * lda + e % n] = a_glob[e];
    for (long long idx = tid; idx < nblk; idx += bs) {
      int bb = (int)((sqrtf(8.0f * (float)idx + 1.0f) - 1.0f) * 0.5f);
      while ((long long)bb * (bb + 1) / 2 > idx) --bb;
      while ((long long)(bb + 1) * (bb + 2) / 2 <= idx) ++bb;
      blk[idx] = (int)(idx - (long long)bb * (bb + 1) / 2) | (bb << 16);
    }
  }
  if (tid == 0) s_flag = 0x7fffffff;
  for (int e = tid; e < vn * n; e += blockDim.x) {
    const int rr = e / n, cc = e - rr * n;
    A_::st(vsm + e, (v0 + rr == cc) ? A_::one() : A_::zero());
  }
  auto write_v = [&]() {
    __syncthreads();
    for (int e = tid; e < vn * n; e += blockDim.x) {
      const int rr = e / n, cc = e - rr * n;
      v_out[(size_t)cc * n + v0 + rr] = vsm[e];
    }
  };
  __syncthreads();

  // initial positive-definiteness check (jacobi.cpp:200-201): every CTA
  // evaluates it identically, so all exit together.
  for (int k = tid; k < n; k += bs)
    if (!A_::gt0(LD(AE(k, k)))) atomicMin(&s_flag, k);
  __syncthreads();
  if (s_flag != 0x7fffffff) {
    if (blockIdx.x == 0 && tid == 0) {
      status->status = kNotPositiveDefinite;
      status->index = s_flag + 1;
      status->value = A_::hi(LD(AE(s_flag, s_flag)));
      status->sweeps = 0;
      status->rotations = 0;
    }
    if (vn) write_v();
    return;
  }

  const int gtid = blockIdx.x * bs + tid, gstride = gridDim.x * bs;
  long long rotations = 0;
  double worst = 0.0;
  int sweeps = 0;
  bool converged = false;
  long long g = 0;  // global round counter

  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    // ---- sweep pre-check: if no pair passes the stop test now, this sweep
    // would rotate nothing (A cannot change), i.e. it is the converged
    // detection sweep of jacobi.cpp:256-260 — decided in one parallel pass.
    {
      if (kSmem) {
        if (tid == 0) s_sweep_flag = 0;
        __syncthreads();
      }
      unsigned found = 0;
      const long long npairs = (long long)n * (n - 1) / 2;
      for (long long e = kSmem ? tid : gtid; e < npairs && !found; e += kSmem ? bs : gstride) {
        int j = (int)((sqrtf(8.0f * (float)e + 1.0f) + 1.0f) * 0.5f);
        while ((long long)j * (j - 1) / 2 > e) --j;
        while ((long long)(j + 1) * j / 2 <= e) ++j;
        const int i = (int)(e - (long long)j * (j - 1) / 2);
        found = A_::active(LD(AE(i, i)), LD(AE(j, j)), LD(AE(i, j)), tol) ? 1u : 0u;
      }
      if (kSmem) {
        if (__any_sync(FULL, found) && lane == 0) s_sweep_flag = 1;
        __syncthreads();
        found = s_sweep_flag;
      } else {
        // grid-wide OR through the sweep parity word of the diag buffer tail
        unsigned* flags = reinterpret_cast<unsigned*>(diagbuf + 6 * np);
        if (__any_sync(FULL, found) && lane == 0) atomicOr(&flags[sweep & 1], 1u);
        gsync();
        found = *(volatile unsigned*)&flags[sweep & 1];
        if (blockIdx.x == 0 && tid == 0) flags[(sweep + 1) & 1] = 0;  // reset for the next sweep
      }
      if (!found) {
        ++sweeps;
        converged = true;
        break;
      }
    }
    // round-0 diagonal blocks for the multi-CTA path
    if (!kSmem && sweep == 0) {
      ST* d0 = diagbuf + (g & 1) * 3 * np;
      for (int k = gtid; k < np; k += gstride) {
        int pp, qq;
        rr_pair(n, 0, k, pp, qq);
        if (qq < n) {
          d0[3 * k] = a[(long long)pp * n + pp];
          d0[3 * k + 1] = a[(long long)qq * n + qq];
          d0[3 * k + 2] = a[(long long)qq * n + pp];
        }
      }
      gsync();
    }
    long long rot_sweep = 0;
    worst = 0.0;
    const bool want_ratio = sweep + 1 == max_sweeps;
    for (int r = 0; r < R; ++r, ++g) {
      const bool trace = !kSmem && g_jtrace && sweep == 0 && r < 64 && blockIdx.x == 0 && tid == 0;
      if (trace) g_jtrace[r * 16 + 0] = clock64();
      const int par = (int)(g & 1);
      const int rnext = (r + 1 == R) ? 0 : r + 1;
      const ST* dcur = diagbuf + par * 3 * np;
      ST* dnext = diagbuf + (par ^ 1) * 3 * np;
      // ---- phase 1: all rotations of the round, redundantly in every CTA.
      // Per-warp partial reductions land in w_* slots, combined after the
      // barrier (slots are rewritten only after the phase-2 barrier).
      if (warp < nw_rot) {
        int act_sum = 0, bad = 0x7fffffff;
        double wmax = 0.0;
        const int kend = min(np, (cr + 1) * rchunk);  // this CTA's slots (all of them without clusters)
        for (int k0 = cr * rchunk; k0 < kend; k0 += bs) {  // uniform trip count within the warp
          const int k = k0 + tid;
          int pp = 0, qq = n;
          if (k < kend) rr_pair(n, r, k, pp, qq);
          AT app = A_::one(), aqq = A_::one(), apq = A_::zero();
          if (qq < n) {
            if (kSmem) {
              app = LD(AE(pp, pp));
              aqq = LD(AE(qq, qq));
              apq = LD(AE(pp, qq));
            } else {
              app = A_::ldg(dcur + 3 * k);
              aqq = A_::ldg(dcur + 3 * k + 1);
              apq = A_::ldg(dcur + 3 * k + 2);
            }
          }
          const bool act = qq < n && A_::active(app, aqq, apq, tol);
          if (want_ratio && qq < n) wmax = fmax(wmax, A_::ratio(app, aqq, apq));
          AT c = A_::one(), s = A_::zero(), npp = app, nqq = aqq;
          if (__any_sync(FULL, act)) {
            AT c2, s2, np2, nq2;
            // inactive lanes rotate a harmless dummy block and discard it
            A_::rotate(act ? app : A_::one(), act ? aqq : A_::one(), act ? apq : A_::one(), c2, s2, np2, nq2);
            if (act) {
              c = c2;
              s = s2;
              npp = np2;
              nqq = nq2;
              if (!A_::gt0(npp)) bad = min(bad, pp);
              if (!A_::gt0(nqq)) bad = min(bad, qq);
            }
          }
          act_sum += act ? 1 : 0;
          if (k < kend) {
            const int word = pp | (qq << 15) | ((act ? 1 : 0) << 30);
            rc[k] = c;
            rsn[k] = s;
            rnpp[k] = npp;
            rnqq[k] = nqq;
            pw[k] = word;
#pragma unroll
            for (int t = 0; t < kMaxCs - 1; ++t)
              if (t + 1 < cs) {
                st_cluster(peer(rc + k, t), c);
                st_cluster(peer(rsn + k, t), s);
                st_cluster(peer(rnpp + k, t), npp);
                st_cluster(peer(rnqq + k, t), nqq);
                st_cluster(peer(pw + k, t), word);
              }
          }
        }
        act_sum = warp_sum(act_sum);
        bad = warp_min(bad);
        if (want_ratio) wmax = warp_max(wmax);
        if (lane == 0) {
          const int wslot = cr * nw_rot + warp;
          w_cnt[wslot] = act_sum;
          w_bad[wslot] = bad;
          w_worst[wslot] = wmax;
#pragma unroll
          for (int t = 0; t < kMaxCs - 1; ++t)
            if (t + 1 < cs) {
              st_cluster(peer(&w_cnt[wslot], t), act_sum);
              st_cluster(peer(&w_bad[wslot], t), bad);
              st_cluster(peer(&w_worst[wslot], t), wmax);
            }
        }
      }
      if (!kSmem) {  // round rnext's slot and partner of every player, for emit()
        for (int x = tid; x < n; x += bs) {
          const int s2 = rr_slot(n, rnext, x);
          int pp, qq;
          rr_pair(n, rnext, s2, pp, qq);
          nsl[x] = s2 | ((pp == x ? 0 : 1) << 16);
          npart[x] = pp == x ? qq : pp;
        }
      }
      csync();
      if (trace) g_jtrace[r * 16 + 1] = clock64();
      int cnt = 0, badx = 0x7fffffff;
      for (int w = 0; w < cs * nw_rot; ++w) {
        cnt += w_cnt[w];
        badx = min(badx, w_bad[w]);
        worst = fmax(worst, w_worst[w]);
      }
      if (badx != 0x7fffffff) {  // NotPositiveDefiniteError(pivot, value), jacobi.cpp:242-243
        if (blockIdx.x == 0 && tid == 0) {
          const int x = badx;
          const int k = rr_slot(n, r, x);
          const int pp = pw[k] & 0x7fff;
          status->status = kNotPositiveDefinite;
          status->index = x + 1;
          status->value = A_::hi(x == pp ? rnpp[k] : rnqq[k]);
          status->sweeps = sweeps;
          status->rotations = rotations;
        }
        if (vn) write_v();
        return;
      }
      rot_sweep += cnt;
      rotations += cnt;
      if (blockIdx.x == 0) {
        for (int k = tid; k < np; k += bs) {
          ST* lg = rot_log + 2 * ((long long)g * np + k);
          A_::st(lg, rc[k]);
          A_::st(lg + 1, rsn[k]);
        }
      }
      // ---- phase 2: 2x2 blocks between pairs aa <= bb; each element has
      // exactly one owner. Off-diagonal blocks: column rotation of bb, then
      // row rotation of aa, written to both triangles (exact symmetry).
      if (kSmem) {
        if (cnt != 0) {
          for (long long idx = tid; idx < nblk; idx += bs) {
            const int w = blk[idx];
            const int aa = w & 0xffff, bb = w >> 16;
            const int wa = pw[aa], wb = pw[bb];
            const bool acta = (wa >> 30) & 1, actb = (wb >> 30) & 1;
            if (!acta && !actb) continue;
            const int p0 = wa & 0x7fff, q0 = (wa >> 15) & 0x7fff;
            if (aa == bb) {  // diagonal block (jacobi.cpp:236-241)
              A_::st(AE(p0, p0), rnpp[aa]);
              A_::st(AE(q0, q0), rnqq[aa]);
              A_::st(AE(p0, q0), A_::zero());
              A_::st(AE(q0, p0), A_::zero());
              continue;
            }
            const int k0 = wb & 0x7fff, l0 = (wb >> 15) & 0x7fff;
            if (q0 < n && l0 < n) {
              AT x00 = LD(AE(p0, k0)), x01 = LD(AE(p0, l0)), x10 = LD(AE(q0, k0)), x11 = LD(AE(q0, l0));
              if (actb) {
                const AT cb = rc[bb], sb = rsn[bb];
                const AT y00 = A_::rot_lo(cb, sb, x00, x01), y01 = A_::rot_hi(cb, sb, x00, x01);
                const AT y10 = A_::rot_lo(cb, sb, x10, x11), y11 = A_::rot_hi(cb, sb, x10, x11);
                x00 = y00;
                x01 = y01;
                x10 = y10;
                x11 = y11;
              }
              if (acta) {
                const AT ca = rc[aa], sa = rsn[aa];
                const AT y00 = A_::rot_lo(ca, sa, x00, x10), y10 = A_::rot_hi(ca, sa, x00, x10);
                const AT y01 = A_::rot_lo(ca, sa, x01, x11), y11 = A_::rot_hi(ca, sa, x01, x11);
                x00 = y00;
                x10 = y10;
                x01 = y01;
                x11 = y11;
              }
              A_::st(AE(p0, k0), x00);
              A_::st(AE(k0, p0), x00);
              A_::st(AE(p0, l0), x01);
              A_::st(AE(l0, p0), x01);
              A_::st(AE(q0, k0), x10);
              A_::st(AE(k0, q0), x10);
              A_::st(AE(q0, l0), x11);
              A_::st(AE(l0, q0), x11);
            } else {  // one of the pairs holds the bye of an odd n
              const int rows[2] = {p0, q0}, cols[2] = {k0, l0};
              const int nr = q0 < n ? 2 : 1, nc = l0 < n ? 2 : 1;
              AT x[2][2];
              for (int u = 0; u < 2; ++u)
                for (int v = 0; v < 2; ++v) x[u][v] = (u < nr && v < nc) ? LD(AE(rows[u], cols[v])) : A_::zero();
              if (actb)
                for (int u = 0; u < 2; ++u) {
                  const AT x0 = x[u][0], x1 = x[u][1];
                  x[u][0] = A_::rot_lo(rc[bb], rsn[bb], x0, x1);
                  x[u][1] = A_::rot_hi(rc[bb], rsn[bb], x0, x1);
                }
              if (acta)
                for (int v = 0; v < 2; ++v) {
                  const AT y0 = x[0][v], y1 = x[1][v];
                  x[0][v] = A_::rot_lo(rc[aa], rsn[aa], y0, y1);
                  x[1][v] = A_::rot_hi(rc[aa], rsn[aa], y0, y1);
                }
              for (int u = 0; u < nr; ++u)
                for (int v = 0; v < nc; ++v) {
                  A_::st(AE(rows[u], cols[v]), x[u][v]);
                  A_::st(AE(cols[v], rows[u]), x[u][v]);
                }
            }
          }
        }
        __syncthreads();
        continue;
      }
      // multi-CTA variant: every block is visited so that the entries the
      // next round's rotations read are published to the diag buffer.
      // Store-once symmetric storage: entry (i, j) lives at its upper-triangle
      // position (min, max) (4 stores per 2x2 block instead of 8; the sweep
      // pre-check, the round-0 buffer and the final diagonal read only the
      // upper triangle).
      auto CEg = [&](int i, int j) -> ST* { return i <= j ? AE(i, j) : AE(j, i); };
      auto emit = [&](int x, int y, AT v) {
        const int w = nsl[x];
        if (x == y) {
          A_::st(dnext + 3 * (w & 0xffff) + (w >> 16), v);
        } else if (npart[x] == y) {
          A_::st(dnext + 3 * (w & 0xffff) + 2, v);
        }
      };
      // The thread's blocks are processed with the next off-diagonal block's
      // four entries already loaded (its L2 round trip overlaps this block's
      // rotations); blocks of a round touch disjoint entries, so the early
      // loads see the round's inputs. Same arithmetic per block.
      auto decode = [&](long long idx, int& aa, int& bb) {
        bb = (int)((sqrtf(8.0f * (float)idx + 1.0f) - 1.0f) * 0.5f);
        while ((long long)bb * (bb + 1) / 2 > idx) --bb;
        while ((long long)(bb + 1) * (bb + 2) / 2 <= idx) ++bb;
        aa = (int)(idx - (long long)bb * (bb + 1) / 2);
      };
      // entries of an off-diagonal block (zero outside an odd n's bye)
      auto load_block = [&](int aa, int bb, AT (&x)[2][2]) {
        const int wa = pw[aa], wb = pw[bb];
        const int rows[2] = {wa & 0x7fff, (wa >> 15) & 0x7fff}, cols[2] = {wb & 0x7fff, (wb >> 15) & 0x7fff};
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v)
            x[u][v] = (rows[u] < n && cols[v] < n) ? LD(CEg(rows[u], cols[v])) : A_::zero();
      };
      // fused V: round r's rotations on this CTA's rows of V (the replay's
      // arithmetic: identity rotations skipped, rot_lo / rot_hi per pair),
      // items [w0, w1) of vn * np
      auto v_update = [&](int w0, int w1) {
        // item w = (row rr, slot k) = (w / np, w % np), stepped without divisions
        int rr = (w0 + tid) / np, k = (w0 + tid) - rr * np;
        for (int w = w0 + tid; w < w1; w += bs, rr += vstep_r, k += vstep_k) {
          if (k >= np) {
            k -= np;
            ++rr;
          }
          const AT c = rc[k], sn = rsn[k];
          if (A_::is_identity(c, sn)) continue;
          const int wk = pw[k];
          const int pp = wk & 0x7fff, qq = (wk >> 15) & 0x7fff;
          ST* row = vsm + (size_t)rr * n;
          const AT t1 = A_::lds(row + pp), t2 = A_::lds(row + qq);
          A_::st(row + pp, A_::rot_lo(c, sn, t1, t2));
          A_::st(row + qq, A_::rot_hi(c, sn, t1, t2));
        }
      };
      const int v_items = vn * np;
      // the share of the V update done while the first block's loads are in
      // flight (the block phase is bound by L2 traffic, not fp64 issue); the
      // rest sits between the round barrier's arrive and wait
      const int v_early = (int)((long long)v_items * vsplit / 100) / bs * bs;
      AT xn[2][2];
      int an = 0, bn = 0;
      long long idx = gtid;
      if (idx < nblk) {
        decode(idx, an, bn);
        if (an != bn) load_block(an, bn, xn);
      }
      if (vn) v_update(0, v_early);
      for (; idx < nblk; idx += gstride) {
        const int aa = an, bb = bn;
        AT x[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v) x[u][v] = xn[u][v];
        if (idx + gstride < nblk) {
          decode(idx + gstride, an, bn);
          if (an != bn) load_block(an, bn, xn);
        }
        const int wa = pw[aa];
        const int p0 = wa & 0x7fff, q0 = (wa >> 15) & 0x7fff;
        const bool acta = (wa >> 30) & 1;
        if (aa == bb) {
          if (q0 >= n) {
            emit(p0, p0, LD(AE(p0, p0)));
            continue;
          }
          AT vpp, vqq, vpq;
          if (acta) {
            vpp = rnpp[aa];
            vqq = rnqq[aa];
            vpq = A_::zero();
            A_::st(AE(p0, p0), vpp);
            A_::st(AE(q0, q0), vqq);
            A_::st(AE(p0, q0), vpq);  // p0 < q0: the canonical copy
          } else {
            vpp = LD(AE(p0, p0));
            vqq = LD(AE(q0, q0));
            vpq = LD(AE(p0, q0));
          }
          emit(p0, p0, vpp);
          emit(q0, q0, vqq);
          emit(p0, q0, vpq);
          continue;
        }
        const int wb = pw[bb];
        const int k0 = wb & 0x7fff, l0 = (wb >> 15) & 0x7fff;
        const bool actb = (wb >> 30) & 1;
        const int rows[2] = {p0, q0}, cols[2] = {k0, l0};
        const int nr = q0 < n ? 2 : 1, nc = l0 < n ? 2 : 1;
        ST* e[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v) e[u][v] = CEg(rows[u], cols[v]);
        if (actb) {
          const AT cb = rc[bb], sb = rsn[bb];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const AT x0 = x[u][0], x1 = x[u][1];
            x[u][0] = A_::rot_lo(cb, sb, x0, x1);
            x[u][1] = A_::rot_hi(cb, sb, x0, x1);
          }
        }
        if (acta) {
          const AT ca = rc[aa], sa = rsn[aa];
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const AT y0 = x[0][v], y1 = x[1][v];
            x[0][v] = A_::rot_lo(ca, sa, y0, y1);
            x[1][v] = A_::rot_hi(ca, sa, y0, y1);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            if (u < nr && v < nc) {
              if (acta || actb) A_::st(e[u][v], x[u][v]);
              emit(rows[u], cols[v], x[u][v]);
            }
          }
      }
      if (trace) g_jtrace[r * 16 + 2] = clock64();
      // ---- the round's grid barrier, split: arrive once this CTA's blocks
      // are written, wait after the fused V update - the rows of V live in
      // this CTA's shared memory and need only the round's rotations, so
      // that work (as long as the block updates at n = 1024 dd) hides the
      // barrier's latency (~2.9 k cycles through cg::grid.sync) and the
      // stragglers instead of preceding them.
      garrive();
      if (vn) v_update(v_early, v_items);
      // (cluster-wide at its end: the peer CTAs write the next round's
      // rotations into this CTA's shared memory, which the V update reads)
      gwait();
      if (trace) g_jtrace[r * 16 + 3] = clock64();
    }
    ++sweeps;
    if (rot_sweep == 0) {
      converged = true;
      break;
    }
  }

  if (kSmem) {
    __syncthreads();
    for (long long e = tid; e < (long long)n * n; e += bs) a_glob[e] = a[(e / n) * lda + e % n];
  }
  if (vn) write_v();
  if (blockIdx.x == 0 && tid == 0) {
    status->status = converged ? kOk : kNoConvergence;
    status->index = converged ? 0 : max_sweeps;
    status->value = converged ? 0.0 : worst;
    status->sweeps = sweeps;
    status->rotations = rotations;
    status->rounds = g;
  }
}

// ---------------------------------------------------------------------------
// Single-CTA Jacobi for matrices resident in shared memory, warp-specialised
// so the latency of the rotation formulas overlaps the 2x2 block updates:
//
//   rotation warps (R):  wait B2(r-1) -> rotations of round r -> arrive B1(r)
//   update warps   (U):  wait B1(r) -> pass 1: the blocks holding the entries
//                        round r+1's rotations read (its diagonal blocks'
//                        images) -> arrive B2(r) -> pass 2: all other blocks
//                        -> U-only barrier B3
//
// so a round costs ~max(rotation latency, block updates) instead of their
// sum. Named barriers: 1 = B1, 2 = B2, 3 = B3 (U only), 4 = R-only.
__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

constexpr int kUpdateWarps = 12;
constexpr int kRotWarps = 4;

__device__ int g_jexp = 0;  // experiment switches (MPSVD_JACOBI_EXP, timing only): 2 skip the bulk, 4 the priority blocks

// partner of x in `round` (n itself for the bye of an odd n)
__device__ __forceinline__ int rr_partner(int n, int round, int x) {
  int pp, qq;
  rr_pair(n, round, rr_slot(n, round, x), pp, qq);
  return pp == x ? qq : pp;
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
constexpr unsigned long long kProgressDone = 1ull << 63;

// Fused V replay CTA: owns `rows` rows of V (shared memory), applies every
// round the solver CTA has published (progress word, release/acquire), and
// writes its rows once the solver reports completion. The rows of V never
// mix, so the replay overlaps the solve instead of following it.
template <typename ST>
__device__ void replay_consumer(const ST* __restrict__ rot_log, int n, DevStatus* status, ST* __restrict__ v_out,
                                int rows, ST* vr) {
  using A_ = Arith<ST>;
  using AT = typename A_::AT;
  const int N = n + (n & 1), np = N / 2, R = N - 1;
  const int row0 = (blockIdx.x - 1) * rows;
  const int nrows = min(rows, n - row0);
  if (nrows <= 0) return;
  const int tid = threadIdx.x, bs = blockDim.x;
  __shared__ unsigned long long s_prog;
  for (int e = tid; e < nrows * n; e += bs) {
    const int rr = e / n, cc = e - rr * n;
    A_::st(vr + e, (row0 + rr == cc) ? A_::one() : A_::zero());
  }
  long long g = 0;
  int r = 0;
  const int items = nrows * np;
  while (true) {
    if (tid == 0) {
      unsigned long long p;
      while (true) {
        p = ld_acquire_u64(&status->progress);
        if ((long long)(p & ~kProgressDone) > g || (p & kProgressDone)) break;
        __nanosleep(64);
      }
      s_prog = p;
    }
    __syncthreads();
    const unsigned long long p = s_prog;
    const long long avail = (long long)(p & ~kProgressDone);
    for (; g < avail; ++g) {
      const ST* lg = rot_log + 2 * g * np;
      for (int w = tid; w < items; w += bs) {
        const int rr = w / np, k = w - rr * np;
        const AT c = A_::ldg(lg + 2 * k), s = A_::ldg(lg + 2 * k + 1);
        if (A_::is_identity(c, s)) continue;
        int pp, qq;
        rr_pair(n, r, k, pp, qq);
        ST* row = vr + (size_t)rr * n;
        const AT t1 = A_::lds(row + pp), t2 = A_::lds(row + qq);
        A_::st(row + pp, A_::rot_lo(c, s, t1, t2));
        A_::st(row + qq, A_::rot_hi(c, s, t1, t2));
      }
      __syncthreads();
      if (++r == R) r = 0;
    }
    if (p & kProgressDone) break;
    __syncthreads();  // s_prog is rewritten only after every thread read it
  }
  for (int e = tid; e < nrows * n; e += bs) {
    const int rr = e / n, cc = e - rr * n;
    v_out[(size_t)cc * n + row0 + rr] = vr[e];
  }
}

template <typename ST, int kNT = 512>
__global__ void __launch_bounds__(kNT, 1)
jacobi_smem(ST* __restrict__ a_glob, ST* __restrict__ rot_log, int n, double tol, int max_sweeps,
            DevStatus* __restrict__ status, ST* __restrict__ v_out, int cons_rows) {
  using A_ = Arith<ST>;
  using AT = typename A_::AT;
  extern __shared__ __align__(16) unsigned char jsm[];
  if (blockIdx.x > 0) {  // fused V replay (cooperative launch: all CTAs co-resident)
    replay_consumer<ST>(rot_log, n, status, v_out, cons_rows, reinterpret_cast<ST*>(jsm));
    return;
  }
  const int N = n + (n & 1), np = N / 2, Rr = N - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool fused = v_out != nullptr;
  unsigned long long* const progress = &status->progress;
  // 16 warps. Warps 0, 4, 8, 12 (scheduler partition 0, warp % 4 == 0) are
  // the rotation warps: the latency-critical rotation chain gets a scheduler
  // and an fp64 pipe of its own; the 12 update warps fill partitions 1-3.
  const int nw_rot = (int)(blockDim.x / 128);  // one rotation warp per 4 warps
  const int NT = blockDim.x, n_rot = 32 * nw_rot, n_upd = NT - n_rot;
  const bool is_rot = (warp & 3) == 0;
  const int wr = warp >> 2, rtid = wr * 32 + lane;  // rotation-warp / rotation-thread index
  unsigned long long* const jt = g_jtrace;  // read once: a global load per use would be timed too
  const int jexp = g_jexp;
  const int utid = (warp - (warp >> 2) - 1) * 32 + lane;  // update-thread index
  const int nw_act = (np + 31) / 32;                      // rotation warps with slots (1 or 2)
  const int NB12 = 32 * nw_act + n_upd;                   // participants of B2
  // B1 also releases the publisher warp (the last rotation warp, idle in the
  // solve) that announces each finished round to the fused replay CTAs
  const bool is_pub = fused && is_rot && wr == nw_rot - 1;
  const int NB1 = NB12 + (fused ? 32 : 0);
  // pitch n+2 (even n): the arithmetic progressions of the round-robin
  // schedule ((r+k, r-k+2), (r+k, r+k), ...) then step by an odd number of
  // 8-byte words, i.e. hit distinct banks (n+1 makes (r-k, r+k+2) step by n).
  const int lda = (n | 1) + 1;
  const unsigned FULL = 0xffffffffu;

  ST* a = reinterpret_cast<ST*>(jsm);
  AT* rbase = reinterpret_cast<AT*>(jsm + (size_t)n * lda * sizeof(ST));
  // two round buffers of [c][s][npp][nqq] + pair words
  auto RC = [&](int b) { return rbase + (size_t)b * 4 * np; };
  int* pwb = reinterpret_cast<int*>(rbase + (size_t)8 * np);  // [2][np]
  int* blk = pwb + 2 * np;                                      // idx -> aa | bb << 16
  __shared__ int s_abort, s_bad, s_flag;
  __shared__ int w_cnt[8];
  __shared__ double w_worst[8];
  auto AE = [&](int row, int col) -> ST* { return a + col * lda + row; };
  // Store-once symmetric storage: entry (i, j) lives at its upper-triangle
  // position (min, max); the 2x2 block updates read and write one copy
  // (4 loads + 4 stores instead of 4 + 8 shared-memory accesses).
  auto CE = [&](int i, int j) -> ST* { return i <= j ? a + j * lda + i : a + i * lda + j; };

  for (int e = tid; e < n * n; e += NT) a[(e / n) * lda + e % n] = a_glob[e];
  for (int idx = tid; idx < np * (np + 1) / 2; idx += NT) {
    int bb = (int)((sqrtf(8.0f * (float)idx + 1.0f) - 1.0f) * 0.5f);
    while (bb * (bb + 1) / 2 > idx) --bb;
    while ((bb + 1) * (bb + 2) / 2 <= idx) ++bb;
    blk[idx] = (idx - bb * (bb + 1) / 2) | (bb << 16);
  }
  // priority blocks (diagonal, (k, k+2), (np-2, np-1), (0, 1) for even n)
  int* pri = blk + np * (np + 1) / 2;
  int npri = 0;
  {
    const bool ev = (n & 1) == 0;
    for (int k = 0; k < np; ++k) pri[npri++] = k | (k << 16);
    for (int k = 0; k + 2 < np; ++k) pri[npri++] = k | ((k + 2) << 16);
    if (np >= 2) pri[npri++] = (np - 2) | ((np - 1) << 16);
    if (ev && np >= 3) pri[npri++] = 0 | (1 << 16);
  }
  if (tid == 0) {
    s_abort = 0;
    s_bad = 0x7fffffff;
  }
  __syncthreads();
  // the update warps walk only the non-priority blocks: compact the block
  // table in place (warp 0, ballot ranks; writes never pass the read index)
  __shared__ int s_nnon;
  if (warp == 0) {
    const bool ev = (n & 1) == 0;
    const int nb = np * (np + 1) / 2;
    int cnt = 0;
    for (int base = 0; base < nb; base += 32) {
      const int idx = base + lane;
      int w = 0;
      bool keep = false;
      if (idx < nb) {
        w = blk[idx];
        const int aa = w & 0xffff, bb = w >> 16;
        keep = !(bb == aa || bb == aa + 2 || (bb == aa + 1 && (aa == np - 2 || (ev && aa == 0))));
      }
      const unsigned m = __ballot_sync(FULL, keep);
      __syncwarp();
      if (keep) blk[cnt + __popc(m & ((1u << lane) - 1))] = w;
      cnt += __popc(m);
      __syncwarp();
    }
    if (lane == 0) s_nnon = cnt;
  }
  __syncthreads();
  const int nnon = s_nnon;
  for (int k = tid; k < n; k += NT)
    if (!A_::gt0(A_::lds(AE(k, k)))) atomicMin(&s_bad, k);
  __syncthreads();
  if (s_bad != 0x7fffffff) {  // jacobi.cpp:200-201
    if (tid == 0) {
      status->status = kNotPositiveDefinite;
      status->index = s_bad + 1;
      status->value = A_::hi(A_::lds(AE(s_bad, s_bad)));
      status->sweeps = 0;
      status->rotations = 0;
      status->rounds = 0;
      if (fused) {
        __threadfence();
        st_release_u64(progress, kProgressDone);
      }
    }
    return;
  }

  long long rotations = 0, g = 0;
  int sweeps = 0;
  bool converged = false;
  double worst = 0.0;

  // one 2x2 block update (pairs aa < bb, or the diagonal block aa == bb)
  auto update_block = [&](int aa, int bb, const AT* rb, const int* pw) {
    const int wa = pw[aa], wb = pw[bb];
    const bool acta = (wa >> 30) & 1, actb = (wb >> 30) & 1;
    if (!acta && !actb) return;
    const AT* rcs = rb;
    const AT* rss = rb + np;
    const int p0 = wa & 0x7fff, q0 = (wa >> 15) & 0x7fff;
    if (aa == bb) {  // jacobi.cpp:236-241
      A_::st(AE(p0, p0), rb[2 * np + aa]);
      A_::st(AE(q0, q0), rb[3 * np + aa]);
      A_::st(AE(p0, q0), A_::zero());  // p0 < q0: the canonical copy
      return;
    }
    const int k0 = wb & 0x7fff, l0 = (wb >> 15) & 0x7fff;
    if (q0 < n && l0 < n) {
      ST* const e00 = CE(p0, k0);
      ST* const e01 = CE(p0, l0);
      ST* const e10 = CE(q0, k0);
      ST* const e11 = CE(q0, l0);
      AT x00 = A_::lds(e00), x01 = A_::lds(e01), x10 = A_::lds(e10), x11 = A_::lds(e11);
      if (actb) {
        const AT cb = rcs[bb], sb = rss[bb];
        const AT y00 = A_::rot_lo(cb, sb, x00, x01), y01 = A_::rot_hi(cb, sb, x00, x01);
        const AT y10 = A_::rot_lo(cb, sb, x10, x11), y11 = A_::rot_hi(cb, sb, x10, x11);
        x00 = y00;
        x01 = y01;
        x10 = y10;
        x11 = y11;
      }
      if (acta) {
        const AT ca = rcs[aa], sa = rss[aa];
        const AT y00 = A_::rot_lo(ca, sa, x00, x10), y10 = A_::rot_hi(ca, sa, x00, x10);
        const AT y01 = A_::rot_lo(ca, sa, x01, x11), y11 = A_::rot_hi(ca, sa, x01, x11);
        x00 = y00;
        x10 = y10;
        x01 = y01;
        x11 = y11;
      }
      A_::st(e00, x00);
      A_::st(e01, x01);
      A_::st(e10, x10);
      A_::st(e11, x11);
      return;
    }
    // a pair holding the bye of an odd n: 1x2 / 2x1 / 1x1 block
    const int rows[2] = {p0, q0}, cols[2] = {k0, l0};
    const int nr = q0 < n ? 2 : 1, nc = l0 < n ? 2 : 1;
    AT x[2][2];
    for (int u = 0; u < 2; ++u)
      for (int v = 0; v < 2; ++v) x[u][v] = (u < nr && v < nc) ? A_::lds(CE(rows[u], cols[v])) : A_::zero();
    if (actb)
      for (int u = 0; u < 2; ++u) {
        const AT x0 = x[u][0], x1 = x[u][1];
        x[u][0] = A_::rot_lo(rcs[bb], rss[bb], x0, x1);
        x[u][1] = A_::rot_hi(rcs[bb], rss[bb], x0, x1);
      }
    if (acta)
      for (int v = 0; v < 2; ++v) {
        const AT y0 = x[0][v], y1 = x[1][v];
        x[0][v] = A_::rot_lo(rcs[aa], rss[aa], y0, y1);
        x[1][v] = A_::rot_hi(rcs[aa], rss[aa], y0, y1);
      }
    for (int u = 0; u < nr; ++u)
      for (int v = 0; v < nc; ++v) {
        A_::st(CE(rows[u], cols[v]), x[u][v]);
      }
  };

  // Two off-diagonal blocks at once (the bulk update's common case): within a
  // round the blocks touch disjoint entries, so both blocks' loads are
  // issued before either block's stores and the two dependent chains
  // (pair words -> entries -> two rotations -> stores) overlap; the
  // arithmetic of each block is update_block's. Blocks that are diagonal,
  // hold an odd n's bye or are fully inactive go through update_block.
  auto full_block = [&](int aa, int bb, const int* pw) {
    const int wa = pw[aa], wb = pw[bb];
    return aa != bb && ((wa | wb) >> 30 & 1) && ((wa >> 15) & 0x7fff) < n && ((wb >> 15) & 0x7fff) < n;
  };
  auto update_pair = [&](int w1, int w2, const AT* rb, const int* pw) {
    const int a1 = w1 & 0xffff, b1 = w1 >> 16, a2 = w2 & 0xffff, b2 = w2 >> 16;
    if (!full_block(a1, b1, pw) || !full_block(a2, b2, pw)) {
      update_block(a1, b1, rb, pw);
      update_block(a2, b2, rb, pw);
      return;
    }
    const AT* rcs = rb;
    const AT* rss = rb + np;
    const int wa1 = pw[a1], wb1 = pw[b1], wa2 = pw[a2], wb2 = pw[b2];
    ST* const e00 = CE(wa1 & 0x7fff, wb1 & 0x7fff);
    ST* const e01 = CE(wa1 & 0x7fff, (wb1 >> 15) & 0x7fff);
    ST* const e10 = CE((wa1 >> 15) & 0x7fff, wb1 & 0x7fff);
    ST* const e11 = CE((wa1 >> 15) & 0x7fff, (wb1 >> 15) & 0x7fff);
    ST* const f00 = CE(wa2 & 0x7fff, wb2 & 0x7fff);
    ST* const f01 = CE(wa2 & 0x7fff, (wb2 >> 15) & 0x7fff);
    ST* const f10 = CE((wa2 >> 15) & 0x7fff, wb2 & 0x7fff);
    ST* const f11 = CE((wa2 >> 15) & 0x7fff, (wb2 >> 15) & 0x7fff);
    AT x00 = A_::lds(e00), x01 = A_::lds(e01), x10 = A_::lds(e10), x11 = A_::lds(e11);
    AT z00 = A_::lds(f00), z01 = A_::lds(f01), z10 = A_::lds(f10), z11 = A_::lds(f11);
    if ((wb1 >> 30) & 1) {
      const AT cb = rcs[b1], sb = rss[b1];
      const AT y00 = A_::rot_lo(cb, sb, x00, x01), y01 = A_::rot_hi(cb, sb, x00, x01);
      const AT y10 = A_::rot_lo(cb, sb, x10, x11), y11 = A_::rot_hi(cb, sb, x10, x11);
      x00 = y00;
      x01 = y01;
      x10 = y10;
      x11 = y11;
    }
    if ((wb2 >> 30) & 1) {
      const AT cb = rcs[b2], sb = rss[b2];
      const AT y00 = A_::rot_lo(cb, sb, z00, z01), y01 = A_::rot_hi(cb, sb, z00, z01);
      const AT y10 = A_::rot_lo(cb, sb, z10, z11), y11 = A_::rot_hi(cb, sb, z10, z11);
      z00 = y00;
      z01 = y01;
      z10 = y10;
      z11 = y11;
    }
    if ((wa1 >> 30) & 1) {
      const AT ca = rcs[a1], sa = rss[a1];
      const AT y00 = A_::rot_lo(ca, sa, x00, x10), y10 = A_::rot_hi(ca, sa, x00, x10);
      const AT y01 = A_::rot_lo(ca, sa, x01, x11), y11 = A_::rot_hi(ca, sa, x01, x11);
      x00 = y00;
      x10 = y10;
      x01 = y01;
      x11 = y11;
    }
    if ((wa2 >> 30) & 1) {
      const AT ca = rcs[a2], sa = rss[a2];
      const AT y00 = A_::rot_lo(ca, sa, z00, z10), y10 = A_::rot_hi(ca, sa, z00, z10);
      const AT y01 = A_::rot_lo(ca, sa, z01, z11), y11 = A_::rot_hi(ca, sa, z01, z11);
      z00 = y00;
      z10 = y10;
      z01 = y01;
      z11 = y11;
    }
    A_::st(e00, x00);
    A_::st(e01, x01);
    A_::st(e10, x10);
    A_::st(e11, x11);
    A_::st(f00, z00);
    A_::st(f01, z01);
    A_::st(f10, z10);
    A_::st(f11, z11);
  };

  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    // sweep pre-check (see jacobi_kernel): nothing passes the stop test ->
    // this sweep is the rotation-free detection sweep
    if (tid == 0) s_flag = 0;
    __syncthreads();
    {
      unsigned found = 0;
      const int npairs = n * (n - 1) / 2;
      for (int e = tid; e < npairs && !found; e += NT) {
        int j = (int)((sqrtf(8.0f * (float)e + 1.0f) + 1.0f) * 0.5f);
        while (j * (j - 1) / 2 > e) --j;
        while ((j + 1) * j / 2 <= e) ++j;
        const int i = e - j * (j - 1) / 2;
        found = A_::active(A_::lds(AE(i, i)), A_::lds(AE(j, j)), A_::lds(AE(i, j)), tol) ? 1u : 0u;
      }
      if (__any_sync(FULL, found) && lane == 0) s_flag = 1;
    }
    __syncthreads();
    if (!s_flag) {
      ++sweeps;
      converged = true;
      break;
    }
    const bool want_ratio = sweep + 1 == max_sweeps;
    const bool even_n = (n & 1) == 0;
    // priority blocks: the blocks of a round that hold every entry the next
    // round's rotations read (the same slot pairs in every round of the
    // circle schedule; tests/test_schedule.py checks this exhaustively)
    auto priority = [&](int aa, int bb) {
      return bb == aa || bb == aa + 2 || (bb == aa + 1 && (aa == np - 2 || (even_n && aa == 0)));
    };
    if (is_rot) {
      // ===== rotation warps: rot(r) -> [U finished round r-1] -> release U
      // for round r -> the priority blocks of round r (which feed rot(r+1)),
      // shared by every rotation warp but the publisher, so the rotation
      // chain never waits for the bulk update. (Carrying each slot's next
      // inputs in registers, with each slot thread updating "its" priority
      // block, was slower: the per-thread block chain sits on the critical
      // path, 2.37 k vs 2.16 k cycles per round at n = 64.)
      long long cnt_sweep = 0;
      double wmax = 0.0;
      bool aborted = false;
      const int n_prio_w = nw_rot - (fused ? 1 : 0);
      const int NPR = 32 * n_prio_w;
      if (wr < n_prio_w) {
        const bool rot_warp = wr < nw_act;
        for (int r = 0; r < Rr; ++r) {
          const bool trace = jt && sweep == 0 && r < 64 && rtid == 0;
          if (trace) jt[r * 16 + 0] = clock64();
          AT* rb = RC((int)((g + r) & 1));
          int* pw = pwb + ((g + r) & 1) * np;
          if (rot_warp) {
            const int k = rtid;  // one slot per rotation thread (np <= 64 here)
            int bad = 0x7fffffff, act_i = 0;
            if (k < np) {
              int pp, qq;
              rr_pair(n, r, k, pp, qq);
              AT app = A_::one(), aqq = A_::one(), apq = A_::zero();
              if (qq < n) {
                app = A_::lds(AE(pp, pp));
                aqq = A_::lds(AE(qq, qq));
                apq = A_::lds(AE(pp, qq));
              }
              const bool act = qq < n && A_::active(app, aqq, apq, tol);
              if (want_ratio && qq < n) wmax = fmax(wmax, A_::ratio(app, aqq, apq));
              AT c = A_::one(), s = A_::zero(), npp = app, nqq = aqq;
              {
                // evaluated for every slot, concurrently with the stop test,
                // and kept only for active pairs (same operations, same inputs)
                AT c2, s2, np2, nq2;
                A_::rotate(app, aqq, apq, c2, s2, np2, nq2);
                if (act) {
                  c = c2;
                  s = s2;
                  npp = np2;
                  nqq = nq2;
                  if (!A_::gt0(npp)) bad = min(bad, pp);
                  if (!A_::gt0(nqq)) bad = min(bad, qq);
                }
              }
              act_i = act ? 1 : 0;
              rb[k] = c;
              rb[np + k] = s;
              rb[2 * np + k] = npp;
              rb[3 * np + k] = nqq;
              pw[k] = pp | (qq << 15) | (act_i << 30);
              ST* lg = rot_log + 2 * ((g + r) * np + k);
              A_::st(lg, c);
              A_::st(lg + 1, s);
            }
            cnt_sweep += __popc(__ballot_sync(FULL, act_i));
            if (__any_sync(FULL, bad != 0x7fffffff)) bad = warp_min(bad);
            if (nw_act > 1) {
              if (lane == 0 && bad != 0x7fffffff) atomicMin(&s_bad, bad);
              nbar_sync(4, 32 * nw_act);
              bad = s_bad;
            }
            if (trace) jt[r * 16 + 1] = clock64();
            if (r > 0) nbar_sync(3, NB12);  // the update warps finished round r-1
            if (trace) jt[r * 16 + 2] = clock64();
            if (bad != 0x7fffffff && rtid == 0) {
              const int kk = rr_slot(n, r, bad);
              const int pp = pw[kk] & 0x7fff;
              status->status = kNotPositiveDefinite;
              status->index = bad + 1;
              status->value = A_::hi(bad == pp ? rb[2 * np + kk] : rb[3 * np + kk]);
              status->sweeps = sweeps;
              status->rotations = rotations;
              status->rounds = g + r;
              s_abort = 1;
            }
            if (bad != 0x7fffffff) __syncwarp();
            nbar_arrive(1, NB1);  // round r's rotations are published (or the abort)
          }
          nbar_sync(5, NPR);  // rb / pw (and s_abort) visible to every priority thread
          if (s_abort) {
            aborted = true;
            break;
          }
          for (int j = (jexp & 4) ? npri : rtid; j < npri; j += NPR) {  // experiment: skip
            const int w = pri[j];
            update_block(w & 0xffff, w >> 16, rb, pw);
          }
          nbar_sync(5, NPR);  // rot(r+1) reads the priority blocks
          if (trace) jt[r * 16 + 3] = clock64();
        }
        if (rot_warp && !aborted) nbar_sync(3, NB12);  // the update warps finished the last round
      }
      if (is_pub) {  // publisher: round g+r's log entries are complete after B1
        for (int r = 0; r < Rr; ++r) {
          nbar_sync(1, NB1);
          if (s_abort) break;
          if (lane == 0) {
            __threadfence();
            st_release_u64(progress, (unsigned long long)(g + r + 1));
          }
        }
      }
      const double wm = want_ratio ? warp_max(wmax) : 0.0;
      if (lane == 0) {
        w_cnt[wr] = (int)cnt_sweep;
        w_worst[wr] = wm;
      }
    } else {
      // ===== update warps: every non-priority block of round r, once round
      // r's rotations are published (B1); done -> B3
      for (int r = 0; r < Rr; ++r) {
        nbar_sync(1, NB1);
        const bool trace = jt && sweep == 0 && r < 64 && utid == 0;
        if (trace) jt[r * 16 + 4] = clock64();
        if (s_abort) break;
        const int b = (int)((g + r) & 1);
        const AT* rb = RC(b);
        const int* pw = pwb + b * np;
        int j = (jexp & 2) ? nnon : utid;  // experiment: skip the bulk update
        if constexpr (sizeof(ST) == sizeof(double))  // fp64 only: the dd pair path spills
          for (; j + n_upd < nnon; j += 2 * n_upd) update_pair(blk[j], blk[j + n_upd], rb, pw);
        for (; j < nnon; j += n_upd) {
          const int w = blk[j];
          update_block(w & 0xffff, w >> 16, rb, pw);
        }
        if (trace) jt[r * 16 + 5] = clock64();
        nbar_arrive(3, NB12);
      }
    }
    __syncthreads();
    if (s_abort) {
      if (fused && tid == 0) {
        __threadfence();
        st_release_u64(progress, kProgressDone);
      }
      return;
    }
    long long cnt = 0;
    for (int w = 0; w < nw_rot; ++w) {
      cnt += w_cnt[w];
      worst = fmax(worst, w_worst[w]);
    }
    g += Rr;
    rotations += cnt;
    ++sweeps;
    if (cnt == 0) {
      converged = true;
      break;
    }
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += NT) a_glob[e] = *CE(e % n, e / n);
  if (tid == 0) {
    status->status = converged ? kOk : kNoConvergence;
    status->index = converged ? 0 : max_sweeps;
    status->value = converged ? 0.0 : worst;
    status->sweeps = sweeps;
    status->rotations = rotations;
    status->rounds = g;
    if (fused) {
      __threadfence();
      st_release_u64(progress, kProgressDone | (unsigned long long)g);
    }
  }
}

// ---------------------------------------------------------------------------
// V replay: V = I, then every logged round's rotations applied to V's
// columns (p, q). Each CTA owns `rows` rows of V in shared memory (rows of V
// never mix) and streams the log in batches of rounds.
template <typename ST>
__global__ void __launch_bounds__(kJacobiThreads)
jacobi_replay(const ST* __restrict__ rot_log, int n, int rows_per_cta, int batch,
              const DevStatus* __restrict__ status, ST* __restrict__ v_out) {
  using A_ = Arith<ST>;
  using AT = typename A_::AT;
  extern __shared__ __align__(16) unsigned char rsm[];
  const int N = n + (n & 1), np = N / 2, R = N - 1;
  const int row0 = blockIdx.x * rows_per_cta;
  const int nrows = min(rows_per_cta, n - row0);
  if (nrows <= 0) return;
  ST* vr = reinterpret_cast<ST*>(rsm);      // [rows][n]
  ST* rot = vr + (size_t)rows_per_cta * n;  // [batch][np][2]
  const int tid = threadIdx.x, bs = blockDim.x;
  for (int e = tid; e < nrows * n; e += bs) {
    const int rr = e / n, cc = e - rr * n;
    A_::st(vr + e, (row0 + rr == cc) ? A_::one() : A_::zero());
  }
  const int st = status->status;
  const long long total = (st == kOk || st == kNoConvergence) ? status->rounds : 0;
  __syncthreads();
  const int items = nrows * np;
  for (long long g0 = 0; g0 < total; g0 += batch) {
    const int nb = (int)min((long long)batch, total - g0);
    for (int e = tid; e < nb * np * 2; e += bs) rot[e] = rot_log[g0 * np * 2 + e];
    __syncthreads();
    int r = (int)(g0 % R);
    for (int b = 0; b < nb; ++b) {
      for (int w = tid; w < items; w += bs) {
        const int rr = w / np, k = w - rr * np;
        const AT c = A_::lds(rot + 2 * ((size_t)b * np + k));
        const AT s = A_::lds(rot + 2 * ((size_t)b * np + k) + 1);
        if (A_::is_identity(c, s)) continue;
        int pp, qq;
        rr_pair(n, r, k, pp, qq);
        ST* row = vr + (size_t)rr * n;
        const AT t1 = A_::lds(row + pp), t2 = A_::lds(row + qq);
        A_::st(row + pp, A_::rot_lo(c, s, t1, t2));
        A_::st(row + qq, A_::rot_hi(c, s, t1, t2));
      }
      __syncthreads();
      if (++r == R) r = 0;
    }
  }
  for (int e = tid; e < nrows * n; e += bs) {
    const int rr = e / n, cc = e - rr * n;
    v_out[(size_t)cc * n + row0 + rr] = vr[e];
  }
}

// ---------------------------------------------------------------------------
// Epilogue (jacobi.cpp:280-304 + thinsvd.cpp:81-89,106 + dense.cpp:220-232).
template <typename ST>
__global__ void finish_sort(const ST* __restrict__ a, int n, DevStatus* __restrict__ status,
                            int* __restrict__ perm, double* __restrict__ lam_hi,
                            double* __restrict__ lam_lo, double* __restrict__ sigma,
                            int working_f64) {
  using A_ = Arith<ST>;
  using AT = typename A_::AT;
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0x7fffffff;
  __syncthreads();
  const bool ok = status->status == kOk;
  for (int i = threadIdx.x; i < n && ok; i += blockDim.x) {
    const AT li = A_::ldg(a + (long long)i * n + i);
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const AT lj = A_::ldg(a + (long long)j * n + j);
      bool greater, equal;
      if constexpr (sizeof(ST) == sizeof(double)) {
        greater = lj > li;
        equal = lj == li;
      } else {
        greater = dd_gt(lj, li);
        equal = lj.hi == li.hi && lj.lo == li.lo;
      }
      rank += greater || (equal && j < i);
    }
    perm[rank] = i;
    double sg;
    if constexpr (sizeof(ST) == sizeof(double)) {
      lam_hi[rank] = li;
      if (lam_lo) lam_lo[rank] = 0.0;
      sg = working_f64 ? sqrt(li) : (double)(float)sqrt(li);
    } else {
      lam_hi[rank] = li.hi;
      if (lam_lo) lam_lo[rank] = li.lo;
      const dd sq = dd_sqrt(li);
      sg = working_f64 ? sq.hi : (double)(float)sq.hi;
    }
    sigma[rank] = sg;
    // check_sigma_normal (thinsvd.cpp:22-26): 1/sigma must not overflow
    const bool tiny = working_f64 ? !(sg >= 2.2250738585072014e-308) : !((float)sg >= 1.17549435e-38f);
    if (tiny) atomicMin(&s_bad, rank);
  }
  __syncthreads();
  if (ok && threadIdx.x == 0 && s_bad != 0x7fffffff) {
    status->status = kTinySingularValue;
    status->index = s_bad + 1;
    status->value = sigma[s_bad];
  }
}

// V replay for fp64 and n <= 128: one warp per row of V, the row held in
// registers (lane l owns columns l, l+32, ...); a rotation's partner value
// comes from another lane by shuffle, so rounds need no block barrier.
template <int NC>
__global__ void __launch_bounds__(128)
jacobi_replay_rows(const double2* __restrict__ rot_log, int n, const DevStatus* __restrict__ status,
                   double* __restrict__ v_out) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n) return;  // warp-uniform
  const int N = n + (n & 1), np = N / 2, R = N - 1;
  const unsigned FULL = 0xffffffffu;
  double v[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) v[j] = (lane + 32 * j == row) ? 1.0 : 0.0;
  const int st = status->status;
  const long long total = (st == kOk || st == kNoConvergence) ? status->rounds : 0;
  int r = 0;
#pragma unroll 2
  for (long long g = 0; g < total; ++g) {
    const double2* lg = rot_log + g * np;
    int part[NC], slot[NC];
    bool isp[NC];
    double2 cs[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int col = lane + 32 * j;
      part[j] = n;
      isp[j] = true;
      cs[j] = make_double2(1.0, 0.0);
      if (col < n) {
        slot[j] = rr_slot(n, r, col);
        int pp, qq;
        rr_pair(n, r, slot[j], pp, qq);
        isp[j] = pp == col;
        part[j] = isp[j] ? qq : pp;
        cs[j] = __ldg(lg + slot[j]);
      }
    }
    double vy[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) vy[j] = 0.0;
#pragma unroll
    for (int src = 0; src < NC; ++src) {
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const double t = __shfl_sync(FULL, v[src], part[j] & 31);
        if ((part[j] >> 5) == src) vy[j] = t;
      }
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const double c = cs[j].x, s = cs[j].y;
      if (part[j] < n && !(s == 0.0 && c == 1.0))
        v[j] = isp[j] ? fma(c, v[j], -(s * vy[j])) : fma(s, vy[j], c * v[j]);
    }
    if (++r == R) r = 0;
  }
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const int col = lane + 32 * j;
    if (col < n) v_out[(long long)col * n + row] = v[j];
  }
}

template <typename ST, typename WT>
__global__ void finish_columns(const ST* __restrict__ v, int n, const DevStatus* __restrict__ status,
                               const int* __restrict__ perm, const double* __restrict__ sigma,
                               WT* __restrict__ v_work, WT* __restrict__ w_work,
                               ST* __restrict__ v_full) {
  using A_ = Arith<ST>;
  using AT = typename A_::AT;
  if (status->status != kOk) return;
  const int jj = blockIdx.x;
  const int src = perm[jj];
  const ST* vc = v + (long long)src * n;
  // first index of the largest |v| (ties: lowest row), jacobi.cpp:290-297
  __shared__ double s_hi[32], s_lo[32];
  __shared__ int s_idx[32];
  double bh = -1.0, bl = 0.0;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const AT x = A_::ldg(vc + i);
    double h, l;
    if constexpr (sizeof(ST) == sizeof(double)) {
      h = fabs(x);
      l = 0.0;
    } else {
      const dd ax = dd_abs(x);
      h = ax.hi;
      l = ax.lo;
    }
    if (h > bh || (h == bh && l > bl)) {
      bh = h;
      bl = l;
      bi = i;
    }
  }
  // warp then block argmax
  for (int off = 16; off > 0; off >>= 1) {
    const double oh = __shfl_down_sync(0xffffffffu, bh, off);
    const double ol = __shfl_down_sync(0xffffffffu, bl, off);
    const int oi = __shfl_down_sync(0xffffffffu, bi, off);
    if (oh > bh || (oh == bh && (ol > bl || (ol == bl && oi < bi)))) {
      bh = oh;
      bl = ol;
      bi = oi;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s_hi[wid] = bh;
    s_lo[wid] = bl;
    s_idx[wid] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) / 32;
    for (int w = 1; w < nw; ++w)
      if (s_hi[w] > s_hi[0] || (s_hi[w] == s_hi[0] && (s_lo[w] > s_lo[0] || (s_lo[w] == s_lo[0] && s_idx[w] < s_idx[0])))) {
        s_hi[0] = s_hi[w];
        s_lo[0] = s_lo[w];
        s_idx[0] = s_idx[w];
      }
  }
  __syncthreads();
  const int imax = s_idx[0];
  const bool flip = A_::hi(A_::ldg(vc + imax)) < 0.0;
  const WT sj = (WT)sigma[jj];
  const int ldw = av_ldw(n);
  if (v_full) {  // sorted, sign-fixed V in the higher precision (stage API)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      AT x = A_::ldg(vc + i);
      if (flip) {
        if constexpr (sizeof(ST) == sizeof(double)) x = -x; else x = dd_neg(x);
      }
      A_::st(v_full + (long long)jj * n + i, x);
    }
  }
  if (!v_work) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = A_::hi(A_::ldg(vc + i));  // dd: hi is the RN image
    const WT vw = (WT)(flip ? -x : x);
    v_work[(long long)jj * n + i] = vw;
    // scale_columns(invert): true division; W stored row-major (W^T) for K7
    w_work[(long long)i * ldw + jj] = vw / sj;
  }
}

// ---------------------------------------------------------------------------
size_t jacobi_log_elems(int n, int max_sweeps) {
  const int N = n + (n & 1);
  return (size_t)max_sweeps * (N - 1) * (N / 2) * 2;
}

template <typename ST>
static cudaError_t launch_jacobi_t(int n, double tol, int max_sweeps, const JacobiWorkspace& ws,
                                   int sm_count, cudaStream_t st, bool* fused_replay) {
  if (fused_replay) *fused_replay = false;
  const int N = n + (n & 1), np = N / 2;
  const size_t smem_a = (size_t)n * (n + 1) * sizeof(ST) + (size_t)np * (np + 1) / 2 * sizeof(int);
  const size_t smem_rot = rot_smem_bytes<ST>(np);
  const size_t smem_limit = 200 * 1024;
  ST* a = (ST*)ws.a;
  ST* d = (ST*)ws.diagbuf;
  ST* lg = (ST*)ws.log;
  DevStatus* status = ws.status;
  // zero the two sweep flag words that follow the double-buffered diag blocks
  cudaMemsetAsync(reinterpret_cast<unsigned char*>(ws.diagbuf) + (size_t)6 * np * sizeof(ST), 0, 16, st);
  const size_t smem_pipe = (size_t)n * ((n | 1) + 1) * sizeof(ST) +
                           (size_t)np * (8 * sizeof(typename Arith<ST>::AT) + 2 * sizeof(int)) +
                           ((size_t)np * (np + 1) / 2 + 2 * np) * sizeof(int);
  if (np <= 64 && smem_pipe <= smem_limit) {  // warp-specialised single-CTA solver
    // fp64 with 64 < n: 24 warps (8 more update warps; the n = 128 round is
    // bound by the bulk update, 5 blocks per update thread with 16 warps)
    const bool wide = sizeof(ST) == sizeof(double) && n > 64 && getenv("MPSVD_JACOBI_NARROW") == nullptr;
    auto k = wide ? jacobi_smem<ST, 768> : jacobi_smem<ST, 512>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pipe);
    // 16 warps (__launch_bounds__(512): 128 registers, no spills); fewer via
    // MPSVD_JACOBI_WARPS (a multiple of 4, for experiments)
    static const int warps_env = [] {
      const int w = getenv("MPSVD_JACOBI_WARPS") ? atoi(getenv("MPSVD_JACOBI_WARPS")) : 16;
      return (w >= 8 && w <= 16 && w % 4 == 0) ? w : 16;
    }();
    const int threads = wide ? 768 : 32 * warps_env;
    static const bool trace = getenv("MPSVD_JACOBI_TRACE") != nullptr;
    unsigned long long* tbuf = nullptr;
    if (trace) {
      cudaMalloc(&tbuf, 64 * 16 * sizeof(unsigned long long));
      cudaMemset(tbuf, 0, 64 * 16 * sizeof(unsigned long long));
      cudaMemcpyToSymbol(g_jtrace, &tbuf, sizeof(tbuf));
      const int ex = getenv("MPSVD_JACOBI_EXP") ? atoi(getenv("MPSVD_JACOBI_EXP")) : 0;
      cudaMemcpyToSymbol(g_jexp, &ex, sizeof(ex));
    }
    // CTA 0 solves; CTAs 1.. replay V concurrently (cooperative launch, so
    // every CTA is resident and the consumers' progress polling is safe)
    const int rows = 8, ncons = (n + rows - 1) / rows;
    ST* vout = (ST*)ws.v;
    int nn = n, ms = max_sweeps, rw = rows;
    double tl = tol;
    void* args[] = {&a, &lg, &nn, &tl, &ms, &status, &vout, &rw};
    const cudaError_t le = cudaLaunchCooperativeKernel((const void*)k, dim3(1 + ncons), dim3(threads), args,
                                                       smem_pipe, st);
    if (le != cudaSuccess) return le;
    if (fused_replay) *fused_replay = true;
    if (trace) {
      unsigned long long h[64 * 16];
      cudaStreamSynchronize(st);
      cudaMemcpy(h, tbuf, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long* nul = nullptr;
      cudaMemcpyToSymbol(g_jtrace, &nul, sizeof(nul));
      cudaFree(tbuf);
      // per round (cycles, SM clock): R = rotation warp, U = update warps
      double acc[5] = {0, 0, 0, 0, 0};
      int cnt = 0;
      for (int r = 1; r + 1 < 63 && h[(r + 1) * 16 + 0]; ++r, ++cnt) {
        const unsigned long long* t = h + r * 16;
        acc[0] += (double)(t[16 + 0] - t[0]);  // period (R round start to next)
        acc[1] += (double)(t[1] - t[0]);        // R: rotations
        acc[2] += (double)(t[2] - t[1]);        // R: wait for U's previous round
        acc[3] += (double)(t[3] - t[2]);        // R: priority blocks
        acc[4] += (double)(t[5] - t[4]);        // U: bulk update
      }
      if (cnt)
        fprintf(stderr,
                "[jacobi trace n=%d] period %.0f | R: rotations %.0f, wait U %.0f, priority blocks %.0f | "
                "U: bulk %.0f (cycles/round, %d rounds)\n",
                n, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, cnt);
    }
    return cudaGetLastError();
  }
  if (smem_a + smem_rot <= smem_limit) {
    auto k = jacobi_kernel<ST, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem_a + smem_rot));
    k<<<1, kJacobiThreads, smem_a + smem_rot, st>>>(a, d, lg, n, tol, max_sweeps, status, nullptr, 0, 0);
    return cudaGetLastError();
  }
  auto k = jacobi_kernel<ST, false>;
  const long long nblk = (long long)np * (np + 1) / 2;
  // CTA size: 512 threads on a full grid; a mid-size matrix (fewer blocks
  // than 512 x SMs) spreads over more, smaller CTAs - never fewer threads
  // than rotation slots, so the rotations stay one pass
  // (MPSVD_JACOBI_GRID_THREADS overrides, for experiments)
  int gthreads = kJacobiGridThreads;
  {
    const char* te = getenv("MPSVD_JACOBI_GRID_THREADS");
    const int tv = te ? atoi(te) : 0;
    if (tv >= 64 && tv <= kJacobiGridThreads && tv % 32 == 0) {
      gthreads = tv;
    } else {
      // c3 (n = 256 dd), eigen phase: 512 threads x 17 CTAs 8.2 ms, 256 x 33
      // 7.4 (fused V 7.1), 128 x 65 7.2 (fused V 6.7)
      while (gthreads > 128 && gthreads / 2 >= np && (nblk + gthreads - 1) / gthreads < sm_count) gthreads /= 2;
    }
  }
  long long want = (nblk + gthreads - 1) / gthreads;
  long long grid = (long long)sm_count;  // one CTA per SM (see kJacobiGridThreads)
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  // fused V: each CTA keeps ceil(n / grid) rows of V in shared memory
  // (MPSVD_JACOBI_REPLAY=1 keeps the separate replay)
  int vrows = (int)((n + grid - 1) / grid);
  size_t smem_grid = smem_rot + 16 + (size_t)vrows * n * sizeof(ST);  // + alignment of the V rows
  // fused unless the grid is small (few CTAs would each carry many rows of V
  // per round; the V update sits between the round barrier's arrive and wait)
  if (smem_grid > 200 * 1024 || (4 * grid < sm_count && getenv("MPSVD_JACOBI_FUSE") == nullptr) ||
      getenv("MPSVD_JACOBI_REPLAY") != nullptr) {
    vrows = 0;
    smem_grid = smem_rot;
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_grid);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, gthreads, smem_grid);
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int nn = n, ms = max_sweeps;
  double tl = tol;
  ST* vout = (ST*)ws.v;
  // percent of the fused V update done ahead of the block updates
  // (MPSVD_JACOBI_VSPLIT, default below)
  int vsplit = 0;  // measured on c5: 0, 30, 50, 70 within 1% of each other, 100 slower (the block phase grows by the V time)
  {
    const char* ve = getenv("MPSVD_JACOBI_VSPLIT");
    if (ve && atoi(ve) >= 0 && atoi(ve) <= 100) vsplit = atoi(ve);
  }
  void* args[] = {&a, &d, &lg, &nn, &tl, &ms, &status, &vout, &vrows, &vsplit};
  static const bool trace = getenv("MPSVD_JACOBI_TRACE") != nullptr;
  unsigned long long* tbuf = nullptr;
  if (trace) {
    cudaMalloc(&tbuf, 64 * 16 * sizeof(unsigned long long));
    cudaMemset(tbuf, 0, 64 * 16 * sizeof(unsigned long long));
    cudaMemcpyToSymbol(g_jtrace, &tbuf, sizeof(tbuf));
  }
  // Experiment switch MPSVD_JACOBI_CLUSTER=2|4: clusters of CTAs share each
  // round's rotations (see the kernel). Off by default: measured on c5
  // (n = 1024 dd) the rotation phase is bound by the latency of one rotation
  // chain, not by fp64 issue, so sharing did not shorten it (5.7 k -> 6.0 k
  // cycles) and the cluster barriers cost more (eigen 570 -> 605 ms).
  int csize = 1;
  {
    const char* ce = getenv("MPSVD_JACOBI_CLUSTER");
    const int want_cs = ce ? atoi(ce) : 1;
    if (np >= 256 && (want_cs == 2 || want_cs == 4) && grid % want_cs == 0) {
      cudaLaunchConfig_t qc = {};
      qc.gridDim = dim3((unsigned)grid);
      qc.blockDim = dim3(gthreads);
      qc.dynamicSmemBytes = smem_grid;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = (unsigned)want_cs;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      qc.attrs = qa;
      qc.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)k, &qc) == cudaSuccess &&
          (long long)nclusters * want_cs >= grid)
        csize = want_cs;
      else
        cudaGetLastError();
    }
  }
  cudaError_t le;
  if (csize > 1) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)grid);
    lc.blockDim = dim3(gthreads);
    lc.dynamicSmemBytes = smem_grid;
    lc.stream = st;
    cudaLaunchAttribute la[2];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = (unsigned)csize;
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    la[1].id = cudaLaunchAttributeCooperative;
    la[1].val.cooperative = 1;
    lc.attrs = la;
    lc.numAttrs = 2;
    le = cudaLaunchKernelExC(&lc, (const void*)k, args);
  } else {
    le = cudaLaunchCooperativeKernel((const void*)k, dim3((unsigned)grid), dim3(gthreads), args, smem_grid, st);
  }
  if (le == cudaSuccess && vrows > 0 && fused_replay) *fused_replay = true;
  if (trace) {
    unsigned long long h[64 * 16];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, tbuf, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long* nul = nullptr;
    cudaMemcpyToSymbol(g_jtrace, &nul, sizeof(nul));
    cudaFree(tbuf);
    double acc[4] = {0, 0, 0, 0};
    int cnt = 0;
    for (int r = 1; r + 1 < 63 && h[(r + 1) * 16 + 0]; ++r, ++cnt) {
      const unsigned long long* t = h + r * 16;
      acc[0] += (double)(t[16] - t[0]);
      acc[1] += (double)(t[1] - t[0]);
      acc[2] += (double)(t[2] - t[1]);
      acc[3] += (double)(t[3] - t[2]);
    }
    if (cnt)
      fprintf(stderr,
              "[jacobi multi-CTA trace n=%d grid=%lld cluster=%d] period %.0f | rotations %.0f, block updates %.0f, grid sync %.0f "
              "(cycles/round, %d rounds)\n",
              n, grid, csize, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, cnt);
  }
  return le;
}

cudaError_t launch_jacobi(bool dd_mode, int n, double tol, int max_sweeps, const JacobiWorkspace& ws,
                          int sm_count, cudaStream_t st, bool* fused_replay) {
  return dd_mode ? launch_jacobi_t<double2>(n, tol, max_sweeps, ws, sm_count, st, fused_replay)
                 : launch_jacobi_t<double>(n, tol, max_sweeps, ws, sm_count, st, fused_replay);
}

template <typename ST>
static cudaError_t launch_replay_t(int n, const JacobiWorkspace& ws, cudaStream_t st) {
  const int N = n + (n & 1), np = N / 2;
  // Every CTA streams the whole rotation log, so the log traffic is
  // (CTAs x log bytes): use about one CTA per SM (n = 1024 dd: 7 rows of V
  // per CTA instead of 1 cut the replay from 846 ms to a few tens), and at
  // least ~256 independent rotations per round per CTA.
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  int rows = (256 + np - 1) / np;
  rows = std::max(rows, (n + sms - 1) / sms);
  if (rows > n) rows = n;
  if (rows < 1) rows = 1;
  const size_t budget = 200 * 1024;
  while (rows > 1 && (size_t)rows * n * sizeof(ST) + (size_t)np * 2 * sizeof(ST) > budget) --rows;
  const size_t row_bytes = (size_t)rows * n * sizeof(ST);
  size_t per_round = (size_t)np * 2 * sizeof(ST);
  int batch = row_bytes < budget ? (int)((budget - row_bytes) / per_round) : 1;
  if (batch < 1) batch = 1;
  if (batch > 256) batch = 256;
  const size_t smem = row_bytes + (size_t)batch * per_round;
  auto k = jacobi_replay<ST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = (n + rows - 1) / rows;
  k<<<grid, kJacobiThreads, smem, st>>>((const ST*)ws.log, n, rows, batch, ws.status, (ST*)ws.v);
  return cudaGetLastError();
}

cudaError_t launch_jacobi_replay(bool dd_mode, int n, const JacobiWorkspace& ws, cudaStream_t st) {
  if (!dd_mode && n <= 128) {
    const int grid = (n + 3) / 4;
    const double2* lg = (const double2*)ws.log;
    double* v = (double*)ws.v;
    if (n <= 32)
      jacobi_replay_rows<1><<<grid, 128, 0, st>>>(lg, n, ws.status, v);
    else if (n <= 64)
      jacobi_replay_rows<2><<<grid, 128, 0, st>>>(lg, n, ws.status, v);
    else
      jacobi_replay_rows<4><<<grid, 128, 0, st>>>(lg, n, ws.status, v);
    return cudaGetLastError();
  }
  return dd_mode ? launch_replay_t<double2>(n, ws, st) : launch_replay_t<double>(n, ws, st);
}

cudaError_t launch_finish(bool dd_mode, int n, const JacobiWorkspace& ws, int* perm, double* lambda_hi,
                          double* lambda_lo, double* sigma, void* v_work, void* w_work,
                          int working_f64, cudaStream_t st, void* v_full) {
  const int threads = n < 1024 ? ((n + 31) / 32) * 32 : 1024;
  if (dd_mode) {
    finish_sort<double2><<<1, threads, 0, st>>>((const double2*)ws.a, n, ws.status, perm, lambda_hi,
                                                lambda_lo, sigma, working_f64);
    if (working_f64)
      finish_columns<double2, double><<<n, 256, 0, st>>>((const double2*)ws.v, n, ws.status, perm,
                                                         sigma, (double*)v_work, (double*)w_work, (double2*)v_full);
    else
      finish_columns<double2, float><<<n, 256, 0, st>>>((const double2*)ws.v, n, ws.status, perm,
                                                        sigma, (float*)v_work, (float*)w_work, (double2*)v_full);
  } else {
    finish_sort<double><<<1, threads, 0, st>>>((const double*)ws.a, n, ws.status, perm, lambda_hi,
                                               lambda_lo, sigma, working_f64);
    if (working_f64)
      finish_columns<double, double><<<n, 256, 0, st>>>((const double*)ws.v, n, ws.status, perm, sigma,
                                                        (double*)v_work, (double*)w_work, (double*)v_full);
    else
      finish_columns<double, float><<<n, 256, 0, st>>>((const double*)ws.v, n, ws.status, perm, sigma,
                                                       (float*)v_work, (float*)w_work, (double*)v_full);
  }
  return cudaGetLastError();
}

cudaError_t launch_finish_columns_f64(int n, const double* v, const DevStatus* status, const int* perm,
                                      const double* sigma, void* v_work, void* w_work, int working_f64,
                                      cudaStream_t st) {
  if (working_f64)
    finish_columns<double, double><<<n, 256, 0, st>>>(v, n, status, perm, sigma, (double*)v_work, (double*)w_work,
                                                      (double*)nullptr);
  else
    finish_columns<double, float><<<n, 256, 0, st>>>(v, n, status, perm, sigma, (float*)v_work, (float*)w_work,
                                                     (double*)nullptr);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace mpsvd
