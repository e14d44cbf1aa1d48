// K4 / K5: two-sided Jacobi eigensolver on the n x n Gram matrix, fp64 (K4)
// or double-double (K5), plus the V replay and the sort/sign/sigma epilogue.
//
// Reference semantics: twosided_impl (proj/src/jacobi.cpp:493-569):
//   * skip a pair when |a_ij| <= tol * sqrt(a_ii) * sqrt(a_jj) (the product of
//     square roots, jacobi.cpp:516-522), tol = n*u (jacobi.cpp:579-580);
//   * zeta = (a_jj - a_ii) / (2 a_ij), t = sign(zeta)/(|zeta| + hypot(1, zeta)),
//     c = 1/hypot(1, t), s = c t (jacobi.cpp:524-529);
//   * a_ii -= t a_ij, a_jj += t a_ij, a_ij = 0 exactly, PD re-check
//     (jacobi.cpp:541-548); converged after a sweep without rotations,
//     NoConvergenceError after max_sweeps (jacobi.cpp:561-567);
//   * stable descending sort, V's first largest entry made >= 0
//     (jacobi.cpp:585-609).
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
  static __device__ __forceinline__ AT hyp1(AT z) {
    const double az = fabs(z);
    return az < 0x1p500 ? sqrt(fma(z, z, 1.0)) : az;
  }
  // returns active; fills c, s, t, new diagonal entries; ratio for NoConvergence payload
  static __device__ __forceinline__ bool rotation(AT app, AT aqq, AT apq, double tol, AT& c, AT& s,
                                                  AT& t, AT& npp, AT& nqq, double& ratio) {
    const double thresh = tol * sqrt(app) * sqrt(aqq);
    ratio = fabs(apq) / sqrt(app * aqq);
    c = 1.0;
    s = 0.0;
    t = 0.0;
    npp = app;
    nqq = aqq;
    if (fabs(apq) <= thresh) return false;
    const double zeta = (aqq - app) / (2.0 * apq);
    t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hyp1(zeta));
    c = 1.0 / hyp1(t);
    s = c * t;
    npp = fma(-t, apq, app);
    nqq = fma(t, apq, aqq);
    return true;
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
  static __device__ __forceinline__ bool rotation(AT app, AT aqq, AT apq, double tol, AT& c, AT& s,
                                                  AT& t, AT& npp, AT& nqq, double& ratio) {
    const dd thresh = dd_mul(dd_mul(dd_from(tol), dd_sqrt(app)), dd_sqrt(aqq));
    ratio = fabs(apq.hi) / sqrt(app.hi * aqq.hi);
    c = dd_from(1.0);
    s = dd_from(0.0);
    t = dd_from(0.0);
    npp = app;
    nqq = aqq;
    if (dd_le(dd_abs(apq), thresh)) return false;
    const dd zeta = dd_div(dd_sub(aqq, app), dd_scale2(apq));
    t = dd_div(dd_from(zeta.hi >= 0.0 ? 1.0 : -1.0), dd_add(dd_abs(zeta), dd_hyp1(zeta)));
    c = dd_div(dd_from(1.0), dd_hyp1(t));
    s = dd_mul(c, t);
    const dd tapq = dd_mul(t, apq);
    npp = dd_sub(app, tapq);
    nqq = dd_add(aqq, tapq);
    return true;
  }
};

// ---------------------------------------------------------------------------
constexpr int kJacobiThreads = 256;

template <typename ST>
struct RotSmem {
  typename Arith<ST>::AT* c;
  typename Arith<ST>::AT* s;
  typename Arith<ST>::AT* npp;
  typename Arith<ST>::AT* nqq;
  int* act;
};

template <typename ST>
__host__ __device__ constexpr size_t rot_smem_bytes(int np) {
  return (size_t)np * (4 * sizeof(typename Arith<ST>::AT) + sizeof(int));
}

template <typename ST, bool kSmem>
__global__ void __launch_bounds__(kJacobiThreads)
jacobi_kernel(ST* __restrict__ a_glob, ST* __restrict__ diagbuf, ST* __restrict__ rot_log, int n,
              double tol, int max_sweeps, DevStatus* __restrict__ status) {
  using A_ = Arith<ST>;
  using AT = typename A_::AT;
  extern __shared__ __align__(16) unsigned char jsm[];
  const int N = n + (n & 1), np = N / 2, R = N - 1;
  const int tid = threadIdx.x, bs = blockDim.x;

  // shared memory carve-up
  RotSmem<ST> rs;
  unsigned char* p = jsm;
  ST* a = a_glob;
  if (kSmem) {
    a = reinterpret_cast<ST*>(p);
    p += (size_t)n * n * sizeof(ST);
  }
  rs.c = reinterpret_cast<AT*>(p);
  p += np * sizeof(AT);
  rs.s = reinterpret_cast<AT*>(p);
  p += np * sizeof(AT);
  rs.npp = reinterpret_cast<AT*>(p);
  p += np * sizeof(AT);
  rs.nqq = reinterpret_cast<AT*>(p);
  p += np * sizeof(AT);
  rs.act = reinterpret_cast<int*>(p);
  __shared__ int s_cnt, s_bad;
  __shared__ unsigned long long s_worst;

  auto LD = [&](const ST* q) -> AT { return kSmem ? A_::lds(q) : A_::ldg(q); };
  auto gsync = [&]() {
    if (kSmem)
      __syncthreads();
    else
      cg::this_grid().sync();
  };

  if (kSmem) {
    for (long long e = tid; e < (long long)n * n; e += bs) a[e] = a_glob[e];
    __syncthreads();
  }

  // initial positive-definiteness check (jacobi.cpp:505-506): every CTA
  // evaluates it identically, so all exit together.
  if (tid == 0) s_bad = 0x7fffffff;
  __syncthreads();
  for (int k = tid; k < n; k += bs)
    if (!A_::gt0(LD(a + (long long)k * n + k))) atomicMin(&s_bad, k);
  __syncthreads();
  if (s_bad != 0x7fffffff) {
    if (blockIdx.x == 0 && tid == 0) {
      status->status = kNotPositiveDefinite;
      status->index = s_bad + 1;
      status->value = A_::hi(LD(a + (long long)s_bad * n + s_bad));
      status->sweeps = 0;
      status->rotations = 0;
    }
    return;
  }

  // round-0 diagonal blocks for the multi-CTA path
  if (!kSmem) {
    const int gt = blockIdx.x * bs + tid, gs = gridDim.x * bs;
    for (int k = gt; k < np; k += gs) {
      int pp, qq;
      rr_pair(n, 0, k, pp, qq);
      if (qq < n) {
        ST* d = diagbuf + 3 * k;
        d[0] = a[(long long)pp * n + pp];
        d[1] = a[(long long)qq * n + qq];
        d[2] = a[(long long)qq * n + pp];
      }
    }
    gsync();
  }

  const int gtid = blockIdx.x * bs + tid, gstride = gridDim.x * bs;
  const long long nblk = (long long)np * (np + 1) / 2;
  long long rotations = 0;
  double worst = 0.0;
  int sweeps = 0;
  bool converged = false;
  long long g = 0;  // global round counter

  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    long long rot_sweep = 0;
    worst = 0.0;
    for (int r = 0; r < R; ++r, ++g) {
      const int rnext = (r + 1) % R;
      const ST* dcur = diagbuf + (g & 1) * 3 * np;
      ST* dnext = diagbuf + ((g + 1) & 1) * 3 * np;
      // ---- phase 1: all rotations of the round (redundant per CTA)
      if (tid == 0) {
        s_cnt = 0;
        s_bad = 0x7fffffff;
        s_worst = 0ull;
      }
      __syncthreads();
      for (int k = tid; k < np; k += bs) {
        int pp, qq;
        rr_pair(n, r, k, pp, qq);
        AT c = A_::one(), s = A_::zero(), t = A_::zero(), npp = A_::zero(), nqq = A_::zero();
        int act = 0;
        if (qq < n) {
          AT app, aqq, apq;
          if (kSmem) {
            app = LD(a + (long long)pp * n + pp);
            aqq = LD(a + (long long)qq * n + qq);
            apq = LD(a + (long long)qq * n + pp);
          } else {
            app = A_::ldg(dcur + 3 * k);
            aqq = A_::ldg(dcur + 3 * k + 1);
            apq = A_::ldg(dcur + 3 * k + 2);
          }
          double ratio = 0.0;
          act = A_::rotation(app, aqq, apq, tol, c, s, t, npp, nqq, ratio) ? 1 : 0;
          atomicMax(&s_worst, (unsigned long long)__double_as_longlong(ratio));
          if (act) {
            atomicAdd(&s_cnt, 1);
            if (!A_::gt0(npp)) atomicMin(&s_bad, pp);
            if (!A_::gt0(nqq)) atomicMin(&s_bad, qq);
          }
        }
        rs.c[k] = c;
        rs.s[k] = s;
        rs.npp[k] = npp;
        rs.nqq[k] = nqq;
        rs.act[k] = act;
        (void)t;
      }
      __syncthreads();
      {
        const double w = __longlong_as_double((long long)s_worst);
        if (worst < w) worst = w;
      }
      if (s_bad != 0x7fffffff) {  // NotPositiveDefiniteError(pivot, value), jacobi.cpp:547-548
        if (blockIdx.x == 0 && tid == 0) {
          const int x = s_bad;
          const int k = rr_slot(n, r, x);
          int pp, qq;
          rr_pair(n, r, k, pp, qq);
          status->status = kNotPositiveDefinite;
          status->index = x + 1;
          status->value = A_::hi(x == pp ? rs.npp[k] : rs.nqq[k]);
          status->sweeps = sweeps;
          status->rotations = rotations;
        }
        return;
      }
      rot_sweep += s_cnt;
      rotations += s_cnt;
      if (blockIdx.x == 0) {
        for (int k = tid; k < np; k += bs) {
          ST* lg = rot_log + 2 * ((long long)g * np + k);
          A_::st(lg, rs.c[k]);
          A_::st(lg + 1, rs.s[k]);
        }
      }
      // ---- phase 2: 2x2 blocks between pairs a <= b
      auto emit = [&](int x, int y, AT v) {
        if (kSmem) return;
        const int s2 = rr_slot(n, rnext, x);
        int pp, qq;
        rr_pair(n, rnext, s2, pp, qq);
        if (x == y) {
          A_::st(dnext + 3 * s2 + (pp == x ? 0 : 1), v);
        } else if ((pp == x && qq == y) || (pp == y && qq == x)) {
          A_::st(dnext + 3 * s2 + 2, v);
        }
      };
      for (long long idx = kSmem ? tid : gtid; idx < nblk; idx += kSmem ? bs : gstride) {
        int bb = (int)((sqrt(8.0 * (double)idx + 1.0) - 1.0) * 0.5);
        while ((long long)bb * (bb + 1) / 2 > idx) --bb;
        while ((long long)(bb + 1) * (bb + 2) / 2 <= idx) ++bb;
        const int aa = (int)(idx - (long long)bb * (bb + 1) / 2);
        int p0, q0;
        rr_pair(n, r, aa, p0, q0);
        if (aa == bb) {
          // diagonal block of pair aa (jacobi.cpp:541-546)
          if (q0 >= n) {
            emit(p0, p0, LD(a + (long long)p0 * n + p0));
            continue;
          }
          AT vpp, vqq, vpq;
          if (rs.act[aa]) {
            vpp = rs.npp[aa];
            vqq = rs.nqq[aa];
            vpq = A_::zero();
            A_::st(a + (long long)p0 * n + p0, vpp);
            A_::st(a + (long long)q0 * n + q0, vqq);
            A_::st(a + (long long)q0 * n + p0, vpq);
            A_::st(a + (long long)p0 * n + q0, vpq);
          } else {
            vpp = LD(a + (long long)p0 * n + p0);
            vqq = LD(a + (long long)q0 * n + q0);
            vpq = LD(a + (long long)q0 * n + p0);
          }
          emit(p0, p0, vpp);
          emit(q0, q0, vqq);
          emit(p0, q0, vpq);
          continue;
        }
        int k0, l0;
        rr_pair(n, r, bb, k0, l0);
        const int rows[2] = {p0, q0}, cols[2] = {k0, l0};
        const int nr = q0 < n ? 2 : 1, nc = l0 < n ? 2 : 1;
        const bool acta = rs.act[aa] != 0, actb = rs.act[bb] != 0;
        AT x[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int w = 0; w < 2; ++w)
            x[u][w] = (u < nr && w < nc) ? LD(a + (long long)cols[w] * n + rows[u]) : A_::zero();
        if (actb) {
          const AT cb = rs.c[bb], sb = rs.s[bb];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const AT x0 = x[u][0], x1 = x[u][1];
            x[u][0] = A_::rot_lo(cb, sb, x0, x1);
            x[u][1] = A_::rot_hi(cb, sb, x0, x1);
          }
        }
        if (acta) {
          const AT ca = rs.c[aa], sa = rs.s[aa];
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const AT y0 = x[0][w], y1 = x[1][w];
            x[0][w] = A_::rot_lo(ca, sa, y0, y1);
            x[1][w] = A_::rot_hi(ca, sa, y0, y1);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            if (u < nr && w < nc) {
              if (acta || actb) {
                A_::st(a + (long long)cols[w] * n + rows[u], x[u][w]);
                A_::st(a + (long long)rows[u] * n + cols[w], x[u][w]);
              }
              emit(rows[u], cols[w], x[u][w]);
            }
          }
      }
      gsync();
    }
    ++sweeps;
    if (rot_sweep == 0) {
      converged = true;
      break;
    }
  }

  if (kSmem) {
    for (long long e = tid; e < (long long)n * n; e += bs) a_glob[e] = a[e];
  }
  if (blockIdx.x == 0 && tid == 0) {
    status->status = converged ? kOk : kNoConvergence;
    status->index = converged ? 0 : max_sweeps;
    status->value = converged ? 0.0 : worst;
    status->sweeps = sweeps;
    status->rotations = rotations;
  }
}

// ---------------------------------------------------------------------------
// V replay: V = I, then every logged round's rotations applied to V's
// columns (p, q); each CTA owns a few rows of V in shared memory and streams
// the log in batches of rounds.
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
  ST* vr = reinterpret_cast<ST*>(rsm);                          // [rows][n]
  ST* rot = vr + (size_t)rows_per_cta * n;                      // [batch][np][2]
  const int tid = threadIdx.x, bs = blockDim.x;
  for (int e = tid; e < nrows * n; e += bs) {
    const int rr = e / n, cc = e % n;
    A_::st(vr + e, (row0 + rr == cc) ? A_::one() : A_::zero());
  }
  const int st = status->status;
  const long long total = (st == kOk || st == kNoConvergence) ? (long long)status->sweeps * R : 0;
  __syncthreads();
  for (long long g0 = 0; g0 < total; g0 += batch) {
    const int nb = (int)min((long long)batch, total - g0);
    for (int e = tid; e < nb * np * 2; e += bs) rot[e] = rot_log[g0 * np * 2 + e];
    __syncthreads();
    for (int b = 0; b < nb; ++b) {
      const int r = (int)((g0 + b) % R);
      for (int w = tid; w < nrows * np; w += bs) {
        const int rr = w / np, k = w % np;
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
    }
  }
  for (int e = tid; e < nrows * n; e += bs) {
    const int rr = e / n, cc = e % n;
    v_out[(size_t)cc * n + row0 + rr] = vr[e];
  }
}

// ---------------------------------------------------------------------------
// Epilogue (jacobi.cpp:585-609 + thinsvd.cpp:81-89,106 + dense.cpp:220-232).
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
  // first index of the largest |v| (ties: lowest row), jacobi.cpp:594-603
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
    w_work[(long long)i * n + jj] = vw / sj;
  }
}

// ---------------------------------------------------------------------------
size_t jacobi_log_elems(int n, int max_sweeps) {
  const int N = n + (n & 1);
  return (size_t)max_sweeps * (N - 1) * (N / 2) * 2;
}

template <typename ST>
static cudaError_t launch_jacobi_t(int n, double tol, int max_sweeps, const JacobiWorkspace& ws,
                                   int sm_count, cudaStream_t st) {
  const int N = n + (n & 1), np = N / 2;
  const size_t smem_a = (size_t)n * n * sizeof(ST);
  const size_t smem_rot = rot_smem_bytes<ST>(np);
  const size_t smem_limit = 200 * 1024;
  ST* a = (ST*)ws.a;
  ST* d = (ST*)ws.diagbuf;
  ST* lg = (ST*)ws.log;
  DevStatus* status = ws.status;
  if (smem_a + smem_rot <= smem_limit) {
    auto k = jacobi_kernel<ST, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem_a + smem_rot));
    k<<<1, kJacobiThreads, smem_a + smem_rot, st>>>(a, d, lg, n, tol, max_sweeps, status);
    return cudaGetLastError();
  }
  auto k = jacobi_kernel<ST, false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_rot);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kJacobiThreads, smem_rot);
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const long long nblk = (long long)np * (np + 1) / 2;
  long long want = (nblk + kJacobiThreads - 1) / kJacobiThreads;
  long long grid = (long long)sm_count * (per_sm < 2 ? per_sm : 2);
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  int nn = n, ms = max_sweeps;
  double tl = tol;
  void* args[] = {&a, &d, &lg, &nn, &tl, &ms, &status};
  return cudaLaunchCooperativeKernel((const void*)k, dim3((unsigned)grid), dim3(kJacobiThreads), args,
                                     smem_rot, st);
}

cudaError_t launch_jacobi(bool dd_mode, int n, double tol, int max_sweeps, const JacobiWorkspace& ws,
                          int sm_count, cudaStream_t st) {
  return dd_mode ? launch_jacobi_t<double2>(n, tol, max_sweeps, ws, sm_count, st)
                 : launch_jacobi_t<double>(n, tol, max_sweeps, ws, sm_count, st);
}

template <typename ST>
static cudaError_t launch_replay_t(int n, const JacobiWorkspace& ws, cudaStream_t st) {
  const int N = n + (n & 1), np = N / 2;
  int rows = (n + 147) / 148;
  if (rows < 1) rows = 1;
  const size_t row_bytes = (size_t)rows * n * sizeof(ST);
  const size_t budget = 160 * 1024;
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

}  // namespace dev
}  // namespace mpsvd
