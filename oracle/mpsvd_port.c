/* TEST INFRASTRUCTURE ONLY — see mpsvd_port.h. CPU restatement of the
 * reference hot path (mp_thin_svd, TwoSidedJacobi branch) plus the
 * double-double extension, in plain C. Built by oracle/Makefile with
 * -ffp-contract=off so every multiply/add rounds exactly where the source
 * says (the reference's x86-64 build has no FMA either: proj/CMakeLists.txt:14
 * sets no -march). Where this file calls fma() it does so on purpose, to
 * restate the device kernels' arithmetic (PORT_SEM_DEVICE).
 */
#define _GNU_SOURCE
#include "mpsvd_port.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

enum {
  ST_OK = 0,
  ST_INVALID = 1,
  ST_NPD = 2,
  ST_NOCONV = 3,
  ST_ZERO_COLUMN = 4,
  ST_ZERO_DIVISOR = 5,
  ST_CAST_OVERFLOW = 6,
  ST_TINY_SV = 7,
  ST_INTERNAL = 10
};

static int set_err(port_error* e, int status, int64_t index, double value) {
  if (e) {
    e->status = status;
    e->index = index;
    e->value = value;
  }
  return status;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ======================================================================== */
/* Schedules                                                                */
/* ======================================================================== */

static int64_t next_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

/* make_partition_plan (proj/src/parallel_gram.cpp:57-77): contiguous,
 * balanced row ranges, the first m%blocks blocks one row longer. */
int port_partition_plan(int64_t m, int workers, int64_t blocks, int64_t* ranges,
                        int64_t* nblocks) {
  if (m < 1) return ST_INVALID;
  if (workers < 1 || (int64_t)workers > m) return ST_INVALID;
  if (blocks == 0) blocks = workers == 1 ? 1 : (m < next_pow2(2 * (int64_t)workers) ? m : next_pow2(2 * (int64_t)workers));
  if (blocks < 1 || blocks > m) return ST_INVALID;
  const int64_t base = m / blocks, extra = m % blocks;
  int64_t row = 0;
  for (int64_t b = 0; b < blocks; ++b) {
    const int64_t len = base + (b < extra ? 1 : 0);
    if (ranges) {
      ranges[2 * b] = row;
      ranges[2 * b + 1] = row + len;
    }
    row += len;
  }
  if (nblocks) *nblocks = blocks;
  return ST_OK;
}

/* Parallel round-robin ("circle method") schedule used by the device Jacobi:
 * N = n rounded up to even; player N-1 is fixed and meets `round`, the rest
 * rotate. Round r in [0, N-2], slot k in [0, N/2-1]; every unordered pair
 * meets exactly once per sweep. q == n marks the bye of an odd n. */
void port_rr_pair(int64_t n, int64_t round, int64_t k, int64_t* p, int64_t* q) {
  const int64_t N = n + (n & 1);
  int64_t a, b;
  if (k == 0) {
    a = N - 1;
    b = round;
  } else {
    a = (round + k) % (N - 1);
    b = (round - k + (N - 1)) % (N - 1);
  }
  *p = a < b ? a : b;
  *q = a < b ? b : a;
}

/* ======================================================================== */
/* Gram (proj/src/parallel_gram.cpp:20-32, 265-298)                         */
/* ======================================================================== */

/* block_gram: upper triangle by ascending-k dots from 0, mirrored. */
static void block_gram_f64(const double* a, int64_t m, int64_t n, int64_t r0, int64_t r1,
                           double* out) {
  for (int64_t j = 0; j < n; ++j) {
    const double* cj = a + j * m;
    for (int64_t i = 0; i <= j; ++i) {
      const double* ci = a + i * m;
      double s = 0.0;
      for (int64_t k = r0; k < r1; ++k) s += ci[k] * cj[k];
      out[j * n + i] = s;
      out[i * n + j] = s;
    }
  }
}

typedef struct {
  const double* a;
  int64_t m, n, nb, first, stride;
  const int64_t* ranges;
  double* slots;
} gram_job;

static void* gram_worker(void* arg) {
  gram_job* j = (gram_job*)arg;
  for (int64_t b = j->first; b < j->nb; b += j->stride)
    block_gram_f64(j->a, j->m, j->n, j->ranges[2 * b], j->ranges[2 * b + 1],
                   j->slots + b * j->n * j->n);
  return NULL;
}

int port_partitioned_gram_f64(const double* a, int64_t m, int64_t n, int64_t blocks,
                              double* out) {
  if (n < 1) return ST_INVALID;
  int64_t nb = 0;
  if (port_partition_plan(m, 1, blocks, NULL, &nb) != ST_OK) return ST_INVALID;
  int64_t* ranges = (int64_t*)malloc(sizeof(int64_t) * 2 * nb);
  port_partition_plan(m, 1, blocks, ranges, &nb);
  double* slots = (double*)calloc((size_t)(nb * n * n), sizeof(double));
  if (!slots || !ranges) return ST_INTERNAL;
  /* Blocks run on up to 16 threads; every block's bits are independent of
   * which thread computes it (parallel_gram.cpp:34-53). */
  int nthreads = (int)(nb < 16 ? nb : 16);
  pthread_t th[16];
  gram_job jobs[16];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (gram_job){a, m, n, nb, t, nthreads, ranges, slots};
    pthread_create(&th[t], NULL, gram_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  /* Fixed binary tree over block indices: (0,1),(2,3),... then width x2. */
  for (int64_t width = 1; width < nb; width *= 2)
    for (int64_t i = 0; i + width < nb; i += 2 * width) {
      double* dst = slots + i * n * n;
      const double* src = slots + (i + width) * n * n;
      for (int64_t k = 0; k < n * n; ++k) dst[k] += src[k];
    }
  memcpy(out, slots, sizeof(double) * (size_t)(n * n));
  free(slots);
  free(ranges);
  return ST_OK;
}

int port_partitioned_gram_f32(const float* a, int64_t m, int64_t n, int64_t blocks,
                              double* out) {
  /* cast(A, Higher) (proj/src/dense.cpp:156-161): exact widening. */
  double* ah = (double*)malloc(sizeof(double) * (size_t)(m * n));
  if (!ah) return ST_INTERNAL;
  for (int64_t k = 0; k < m * n; ++k) ah[k] = (double)a[k];
  int st = port_partitioned_gram_f64(ah, m, n, blocks, out);
  free(ah);
  return st;
}

/* ======================================================================== */
/* Two-sided Jacobi, fp64 (proj/src/jacobi.cpp:189-311)                     */
/* ======================================================================== */

/* Stable descending permutation (jacobi.cpp:120-129): insertion sort keeps
 * equal keys in input order. */
static void descending_perm_f64(const double* vals, int64_t n, int64_t* perm) {
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  for (int64_t i = 1; i < n; ++i) {
    int64_t x = perm[i];
    int64_t j = i - 1;
    while (j >= 0 && vals[x] > vals[perm[j]]) {
      perm[j + 1] = perm[j];
      --j;
    }
    perm[j + 1] = x;
  }
}

/* Device-semantics helpers: the exact expressions the CUDA kernels evaluate. */
static inline double rot_lo(double c, double s, double x, double y) { return fma(c, x, -(s * y)); }
static inline double rot_hi(double c, double s, double x, double y) { return fma(s, x, c * y); }

/* finish (jacobi.cpp:280-304): sort by eigenvalue, sign from V's first
 * largest-magnitude entry. */
static void finish_f64(const double* a, const double* v, int64_t n, double* lambda,
                       double* vout) {
  double* lam = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) lam[i] = a[i * n + i];
  descending_perm_f64(lam, n, perm);
  for (int64_t jj = 0; jj < n; ++jj) {
    const int64_t src = perm[jj];
    const double* vc = v + src * n;
    int64_t imax = 0;
    double amax = -1.0;
    for (int64_t i = 0; i < n; ++i)
      if (fabs(vc[i]) > amax) {
        amax = fabs(vc[i]);
        imax = i;
      }
    const double flip = vc[imax] < 0.0 ? -1.0 : 1.0;
    for (int64_t i = 0; i < n; ++i) vout[jj * n + i] = flip * vc[i];
    lambda[jj] = lam[src];
  }
  free(lam);
  free(perm);
}

/* twosided_impl restated (jacobi.cpp:189-264): cyclic by rows. */
static int jacobi_cyclic_f64(double* A, double* V, int64_t n, double tol, int max_sweeps,
                             port_jacobi_stats* st, port_error* err) {
#define AE(i, j) A[(j) * n + (i)]
  const double reltol = tol;
  double worst = 0.0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    worst = 0.0;
    for (int64_t i = 0; i < n - 1; ++i) {
      for (int64_t j = i + 1; j < n; ++j) {
        const double aii = AE(i, i), ajj = AE(j, j), aij = AE(i, j);
        const double thresh = reltol * sqrt(aii) * sqrt(ajj);
        const double ratio = fabs(aij) / sqrt(aii * ajj);
        if (worst < ratio) worst = ratio;
        if (fabs(aij) <= thresh) continue;
        const double zeta = (ajj - aii) / (2.0 * aij);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
        const double cs = 1.0 / hypot(1.0, t);
        const double sn = cs * t;
        for (int64_t k = 0; k < n; ++k) {
          if (k == i || k == j) continue;
          const double aki = AE(k, i), akj = AE(k, j);
          const double ni = cs * aki - sn * akj;
          const double nj = sn * aki + cs * akj;
          AE(k, i) = ni;
          AE(i, k) = ni;
          AE(k, j) = nj;
          AE(j, k) = nj;
        }
        AE(i, i) = aii - t * aij;
        AE(j, j) = ajj + t * aij;
        AE(i, j) = 0.0;
        AE(j, i) = 0.0;
        if (!(AE(i, i) > 0.0)) return set_err(err, ST_NPD, i + 1, AE(i, i));
        if (!(AE(j, j) > 0.0)) return set_err(err, ST_NPD, j + 1, AE(j, j));
        double* vi = V + i * n;
        double* vj = V + j * n;
        for (int64_t k = 0; k < n; ++k) {
          const double t1 = vi[k], t2 = vj[k];
          vi[k] = cs * t1 - sn * t2;
          vj[k] = sn * t1 + cs * t2;
        }
        rotated = 1;
        if (st) ++st->rotations;
      }
    }
    if (st) ++st->sweeps;
    if (!rotated) return ST_OK;
  }
  return set_err(err, ST_NOCONV, max_sweeps, worst);
#undef AE
}

/* Device semantics: parallel round-robin rounds. All rotations of a round
 * are computed from the matrix at the start of the round; every 2x2 block
 * between two pairs a<b gets the column rotation of b first, then the row
 * rotation of a; diagonal blocks take the t*a_pq update (jacobi.cpp:236-241)
 * with fma; V columns are rotated with the same fma forms. */
static int jacobi_rr_f64(double* A, double* V, int64_t n, double tol, int max_sweeps,
                         port_jacobi_stats* st, port_error* err) {
#define AE(i, j) A[(j) * n + (i)]
  const int64_t N = n + (n & 1), np = N / 2;
  int64_t* P = (int64_t*)malloc(sizeof(int64_t) * (size_t)np);
  int64_t* Q = (int64_t*)malloc(sizeof(int64_t) * (size_t)np);
  double* C = (double*)malloc(sizeof(double) * (size_t)np);
  double* S = (double*)malloc(sizeof(double) * (size_t)np);
  double* T = (double*)malloc(sizeof(double) * (size_t)np);
  int* act = (int*)malloc(sizeof(int) * (size_t)np);
  double worst = 0.0;
  int status = ST_NOCONV;
  for (int sweep = 0; sweep < max_sweeps && status == ST_NOCONV; ++sweep) {
    int64_t rot_in_sweep = 0;
    worst = 0.0;
    for (int64_t r = 0; r < N - 1; ++r) {
      for (int64_t k = 0; k < np; ++k) {
        port_rr_pair(n, r, k, &P[k], &Q[k]);
        act[k] = 0;
        C[k] = 1.0;
        S[k] = 0.0;
        T[k] = 0.0;
        if (Q[k] >= n) continue;
        const double aii = AE(P[k], P[k]), ajj = AE(Q[k], Q[k]), aij = AE(P[k], Q[k]);
        /* device formula (jacobi.cu Arith<double>::rotation) */
        const double pr = aii * ajj;
        const double thresh = (pr > 0x1p-1000 && pr < 0x1p1000) ? tol * sqrt(pr) : tol * sqrt(aii) * sqrt(ajj);
        if (sweep + 1 == max_sweeps) {
          const double ratio = fabs(aij) / sqrt(pr);
          if (worst < ratio) worst = ratio;
        }
        if (fabs(aij) <= thresh) continue;
        double x = ajj - aii, y = 2.0 * aij;
        const int xzero = x == 0.0, xpos = x > 0.0;
        const double big = fmax(fabs(x), fabs(y));
        if (!(big < 0x1p500 && big > 0x1p-500)) {
          int e;
          frexp(big, &e);
          x = ldexp(x, -e);
          y = ldexp(y, -e);
        }
        const double ax = fabs(x);
        const double q = fma(x, x, y * y);
        const double r = sqrt(q), iq = 1.0 / q;
        const double den = ax + r;
        const double t = xzero ? 1.0 : (xpos ? y : -y) / den;
        const double c = sqrt(fma(0.5, ax * (r * iq), 0.5));
        C[k] = c;
        S[k] = c * t;
        T[k] = t;
        act[k] = 1;
        ++rot_in_sweep;
      }
      /* off-diagonal 2x2 blocks */
      for (int64_t a = 0; a < np; ++a) {
        for (int64_t b = a + 1; b < np; ++b) {
          if (!act[a] && !act[b]) continue;
          const int64_t rows[2] = {P[a], Q[a]}, cols[2] = {P[b], Q[b]};
          const int nr = Q[a] < n ? 2 : 1, nc = Q[b] < n ? 2 : 1;
          double x[2][2] = {{0, 0}, {0, 0}};
          for (int u = 0; u < nr; ++u)
            for (int w = 0; w < nc; ++w) x[u][w] = AE(rows[u], cols[w]);
          if (act[b])
            for (int u = 0; u < nr; ++u) {
              const double x0 = x[u][0], x1 = x[u][1];
              x[u][0] = rot_lo(C[b], S[b], x0, x1);
              x[u][1] = rot_hi(C[b], S[b], x0, x1);
            }
          if (act[a])
            for (int w = 0; w < nc; ++w) {
              const double y0 = x[0][w], y1 = x[1][w];
              x[0][w] = rot_lo(C[a], S[a], y0, y1);
              x[1][w] = rot_hi(C[a], S[a], y0, y1);
            }
          for (int u = 0; u < nr; ++u)
            for (int w = 0; w < nc; ++w) {
              AE(rows[u], cols[w]) = x[u][w];
              AE(cols[w], rows[u]) = x[u][w];
            }
        }
      }
      /* diagonal blocks + positive-definiteness check (first failing index) */
      int64_t bad_idx = 0;
      double bad_val = 0.0;
      for (int64_t k = 0; k < np; ++k) {
        if (!act[k]) continue;
        const int64_t p = P[k], q = Q[k];
        const double apq = AE(p, q);
        const double app = fma(-T[k], apq, AE(p, p));
        const double aqq = fma(T[k], apq, AE(q, q));
        AE(p, p) = app;
        AE(q, q) = aqq;
        AE(p, q) = 0.0;
        AE(q, p) = 0.0;
        if (!(app > 0.0) && (bad_idx == 0 || p + 1 < bad_idx)) {
          bad_idx = p + 1;
          bad_val = app;
        }
        if (!(aqq > 0.0) && (bad_idx == 0 || q + 1 < bad_idx)) {
          bad_idx = q + 1;
          bad_val = aqq;
        }
      }
      if (bad_idx) {
        status = set_err(err, ST_NPD, bad_idx, bad_val);
        break;
      }
      for (int64_t k = 0; k < np; ++k) {
        if (!act[k]) continue;
        double* vp = V + P[k] * n;
        double* vq = V + Q[k] * n;
        for (int64_t x = 0; x < n; ++x) {
          const double t1 = vp[x], t2 = vq[x];
          vp[x] = rot_lo(C[k], S[k], t1, t2);
          vq[x] = rot_hi(C[k], S[k], t1, t2);
        }
      }
    }
    if (status != ST_NOCONV) break;
    if (st) {
      ++st->sweeps;
      st->rotations += rot_in_sweep;
    }
    if (rot_in_sweep == 0) status = ST_OK;
  }
  if (status == ST_NOCONV) set_err(err, ST_NOCONV, max_sweeps, worst);
  free(P);
  free(Q);
  free(C);
  free(S);
  free(T);
  free(act);
  return status;
#undef AE
}

int port_twosided_jacobi_f64(const double* mtx, int64_t n, double tol, int max_sweeps,
                             int sem, double* lambda, double* v,
                             port_jacobi_stats* stats, port_error* err) {
  set_err(err, ST_OK, 0, 0.0);
  if (n < 1 || max_sweeps < 1) return set_err(err, ST_INVALID, 0, 0.0);
  if (!(tol > 0.0)) tol = (double)n * 0x1p-53; /* jacobi.cpp:274-275 */
  if (stats) {
    stats->sweeps = 0;
    stats->rotations = 0;
    stats->pairs_per_sweep = n * (n - 1) / 2;
  }
  double* A = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* V = (double*)calloc((size_t)(n * n), sizeof(double));
  memcpy(A, mtx, sizeof(double) * (size_t)(n * n));
  for (int64_t i = 0; i < n; ++i) V[i * n + i] = 1.0;
  int st = ST_OK;
  for (int64_t k = 0; k < n; ++k)
    if (!(A[k * n + k] > 0.0)) {
      st = set_err(err, ST_NPD, k + 1, A[k * n + k]);
      break;
    }
  if (st == ST_OK)
    st = sem == PORT_SEM_REFERENCE ? jacobi_cyclic_f64(A, V, n, tol, max_sweeps, stats, err)
                                   : jacobi_rr_f64(A, V, n, tol, max_sweeps, stats, err);
  if (st == ST_OK) finish_f64(A, V, n, lambda, v);
  free(A);
  free(V);
  return st;
}

/* ======================================================================== */
/* One-sided branches of mp_thin_svd (proj/src/thinsvd.cpp:37-47,90-104)     */
/* ======================================================================== */

/* cholesky_impl (proj/src/dense.cpp:39-58), upper factor, strict lower part
 * zero. The device's right-looking K8 applies the same operations to every
 * entry in the same order, so one restatement serves both semantics. */
int port_cholesky_f64(const double* m, int64_t n, double* r, port_error* err) {
  set_err(err, ST_OK, 0, 0.0);
  memset(r, 0, sizeof(double) * (size_t)(n * n));
  for (int64_t k = 0; k < n; ++k) {
    double d = m[k * n + k];
    for (int64_t i = 0; i < k; ++i) {
      const double rik = r[k * n + i];
      d -= rik * rik;
    }
    if (!(d > 0.0)) return set_err(err, ST_NPD, k + 1, d);
    const double rkk = sqrt(d);
    r[k * n + k] = rkk;
    for (int64_t j = k + 1; j < n; ++j) {
      double s = m[j * n + k];
      for (int64_t i = 0; i < k; ++i) s -= r[k * n + i] * r[j * n + i];
      r[j * n + k] = s / rkk;
    }
  }
  return ST_OK;
}

/* One-sided Jacobi cores, generated for float and double.
 *   reference: onesided_impl (proj/src/jacobi.cpp:49-118), cyclic by rows,
 *              make_rotation with hypot (:34-40), scaled_norm_t (:12-28);
 *   device:    K9 (csrc/onesided.cu): round-robin pairs, per-lane fma
 *              partials + xor butterfly, the closed-form rotation, fma
 *              column updates, two-pass max-scaled norms.
 * x: m x n (rotated in place), v: n x n (set to I), sig: n column norms.
 * Returns the status; *worst = the last sweep's worst ratio. */
#define DEFINE_ONESIDED(T, SUF, SQRT, FABS, HYPOT, FMA, FMAX, FREXP, LDEXP, BIG, SMALL)                      \
  static T scaled_norm_ref_##SUF(const T* x, int64_t len) {                                                   \
    T scale = (T)0, ssq = (T)1;                                                                              \
    for (int64_t k = 0; k < len; ++k) {                                                                       \
      if (x[k] != (T)0) {                                                                                    \
        const T ax = FABS(x[k]);                                                                              \
        if (scale < ax) {                                                                                     \
          const T r = scale / ax;                                                                             \
          ssq = (T)1 + ssq * r * r;                                                                           \
          scale = ax;                                                                                         \
        } else {                                                                                              \
          const T r = ax / scale;                                                                             \
          ssq += r * r;                                                                                       \
        }                                                                                                     \
      }                                                                                                       \
    }                                                                                                         \
    return scale * SQRT(ssq);                                                                                 \
  }                                                                                                           \
  static T butterfly_sum_##SUF(T* l) {                                                                        \
    for (int o = 16; o > 0; o >>= 1) {                                                                        \
      T t[32];                                                                                                \
      for (int i = 0; i < 32; ++i) t[i] = l[i] + l[i ^ o];                                                    \
      memcpy(l, t, sizeof(t));                                                                                \
    }                                                                                                         \
    return l[0];                                                                                              \
  }                                                                                                           \
  static void rotate_cols_##SUF(T* xi, T* xj, int64_t len, T cs, T sn, int dev) {                             \
    for (int64_t k = 0; k < len; ++k) {                                                                       \
      const T t1 = xi[k], t2 = xj[k];                                                                         \
      if (dev) {                                                                                              \
        xi[k] = FMA(cs, t1, -(sn * t2));                                                                      \
        xj[k] = FMA(sn, t1, cs * t2);                                                                         \
      } else {                                                                                                \
        xi[k] = cs * t1 - sn * t2;                                                                            \
        xj[k] = sn * t1 + cs * t2;                                                                            \
      }                                                                                                       \
    }                                                                                                         \
  }                                                                                                           \
  /* one pair; returns 1 if rotated, -1/-2 for a zero column i/j */                                           \
  static int pair_##SUF(T* x, T* v, int64_t m, int64_t n, int64_t i, int64_t j, T reltol, int dev,            \
                        double* worst) {                                                                      \
    T* xi = x + i * m;                                                                                        \
    T* xj = x + j * m;                                                                                        \
    T a = (T)0, b = (T)0, c = (T)0;                                                                           \
    if (dev) {                                                                                                \
      T la[32], lb[32], lc[32];                                                                               \
      for (int l = 0; l < 32; ++l) {                                                                         \
        la[l] = lb[l] = lc[l] = (T)0;                                                                         \
        for (int64_t e = l; e < m; e += 32) {                                                                 \
          la[l] = FMA(xi[e], xi[e], la[l]);                                                                   \
          lb[l] = FMA(xj[e], xj[e], lb[l]);                                                                   \
          lc[l] = FMA(xi[e], xj[e], lc[l]);                                                                   \
        }                                                                                                     \
      }                                                                                                       \
      a = butterfly_sum_##SUF(la);                                                                            \
      b = butterfly_sum_##SUF(lb);                                                                            \
      c = butterfly_sum_##SUF(lc);                                                                            \
    } else {                                                                                                  \
      for (int64_t k = 0; k < m; ++k) {                                                                       \
        a += xi[k] * xi[k];                                                                                   \
        b += xj[k] * xj[k];                                                                                   \
        c += xi[k] * xj[k];                                                                                   \
      }                                                                                                       \
    }                                                                                                         \
    if (a == (T)0) return -1;                                                                                 \
    if (b == (T)0) return -2;                                                                                 \
    const T thresh = reltol * SQRT(a) * SQRT(b);                                                              \
    const double ratio = (double)FABS(c) / (sqrt((double)a) * sqrt((double)b));                               \
    if (ratio > *worst) *worst = ratio;                                                                       \
    if (FABS(c) <= thresh) return 0;                                                                          \
    T cs, sn;                                                                                                 \
    if (dev) {                                                                                                \
      const T dx = b - a, dy = (T)2 * c, ax = FABS(dx);                                                       \
      const T big = FMAX(ax, FABS(dy));                                                                       \
      T rr;                                                                                                   \
      if (big < BIG && big > SMALL) {                                                                         \
        rr = SQRT(FMA(dx, dx, dy * dy));                                                                      \
      } else {                                                                                                \
        int e2;                                                                                               \
        FREXP(big, &e2);                                                                                      \
        const T xs = LDEXP(dx, -e2), ys = LDEXP(dy, -e2);                                                     \
        rr = LDEXP(SQRT(FMA(xs, xs, ys * ys)), e2);                                                           \
      }                                                                                                       \
      const T den = ax + rr;                                                                                  \
      const T tt = dx == (T)0 ? (T)1 : (dx > (T)0 ? dy : -dy) / den;                                          \
      cs = sizeof(T) == 4 ? (T)1 / (T)sqrt((double)tt * (double)tt + 1.0) /* K9 OsTraits<float>::cosine */    \
                          : SQRT(den / ((T)2 * rr));                                                          \
      sn = cs * tt;                                                                                           \
    } else {                                                                                                  \
      const T zeta = (b - a) / ((T)2 * c);                                                                    \
      const T t = (zeta >= (T)0 ? (T)1 : (T)-1) / (FABS(zeta) + HYPOT((T)1, zeta));                         \
      cs = (T)1 / HYPOT((T)1, t);                                                                             \
      sn = cs * t;                                                                                            \
    }                                                                                                         \
    rotate_cols_##SUF(xi, xj, m, cs, sn, dev);                                                                \
    rotate_cols_##SUF(v + i * n, v + j * n, n, cs, sn, dev);                                                  \
    return 1;                                                                                                 \
  }                                                                                                           \
  static int onesided_##SUF(T* x, T* v, int64_t m, int64_t n, double tol, int max_sweeps, int dev, T* sig,    \
                            port_jacobi_stats* st, port_error* err) {                                         \
    memset(v, 0, sizeof(T) * (size_t)(n * n));                                                               \
    for (int64_t i = 0; i < n; ++i) v[i * n + i] = (T)1;                                                      \
    const T reltol = (T)tol;                                                                                  \
    double worst = 0.0;                                                                                       \
    int converged = 0, sweep = 0;                                                                             \
    int64_t rotations = 0;                                                                                    \
    const int64_t N = n + (n & 1), np = N / 2;                                                                \
    for (; sweep < max_sweeps; ++sweep) {                                                                     \
      int rotated = 0;                                                                                        \
      int64_t bad = -1;                                                                                       \
      worst = 0.0;                                                                                            \
      if (dev) {                                                                                              \
        for (int64_t r = 0; r < N - 1; ++r)                                                                   \
          for (int64_t k = 0; k < np; ++k) {                                                                  \
            int64_t p, q;                                                                                     \
            port_rr_pair(n, r, k, &p, &q);                                                                    \
            if (q >= n) continue;                                                                             \
            const int res = pair_##SUF(x, v, m, n, p, q, reltol, 1, &worst);                                  \
            if (res < 0) {                                                                                    \
              const int64_t col = res == -1 ? p : q;                                                          \
              if (bad < 0 || col < bad) bad = col;                                                            \
            } else if (res) {                                                                                 \
              rotated = 1;                                                                                    \
              ++rotations;                                                                                    \
            }                                                                                                 \
          }                                                                                                   \
        if (bad >= 0) {                                                                                       \
          if (st) st->sweeps = sweep + 1;                                                                     \
          return set_err(err, ST_ZERO_COLUMN, bad + 1, 0.0);                                                  \
        }                                                                                                     \
      } else {                                                                                                \
        for (int64_t i = 0; i < n - 1; ++i)                                                                   \
          for (int64_t j = i + 1; j < n; ++j) {                                                               \
            const int res = pair_##SUF(x, v, m, n, i, j, reltol, 0, &worst);                                  \
            if (res < 0) return set_err(err, ST_ZERO_COLUMN, (res == -1 ? i : j) + 1, 0.0);                   \
            if (res) {                                                                                        \
              rotated = 1;                                                                                    \
              ++rotations;                                                                                    \
            }                                                                                                 \
          }                                                                                                   \
      }                                                                                                       \
      if (!rotated) {                                                                                         \
        converged = 1;                                                                                        \
        ++sweep;                                                                                              \
        break;                                                                                                \
      }                                                                                                       \
    }                                                                                                         \
    if (st) {                                                                                                 \
      st->sweeps = sweep;                                                                                     \
      st->rotations = rotations;                                                                              \
      st->pairs_per_sweep = n * (n - 1) / 2;                                                                  \
    }                                                                                                         \
    if (!converged) return set_err(err, ST_NOCONV, max_sweeps, worst);                                        \
    for (int64_t j = 0; j < n; ++j) {                                                                         \
      const T* xj = x + j * m;                                                                                \
      T s;                                                                                                    \
      if (dev) {                                                                                              \
        T mx = (T)0;                                                                                          \
        for (int64_t e = 0; e < m; ++e) mx = FMAX(mx, FABS(xj[e]));                                           \
        T l[32];                                                                                              \
        for (int ll = 0; ll < 32; ++ll) {                                                                     \
          l[ll] = (T)0;                                                                                       \
          if (mx > (T)0)                                                                                      \
            for (int64_t e = ll; e < m; e += 32) {                                                            \
              const T y = xj[e] / mx;                                                                         \
              l[ll] = FMA(y, y, l[ll]);                                                                       \
            }                                                                                                 \
        }                                                                                                     \
        s = mx * SQRT(butterfly_sum_##SUF(l));                                                                \
      } else {                                                                                                \
        s = scaled_norm_ref_##SUF(xj, m);                                                                     \
      }                                                                                                       \
      sig[j] = s;                                                                                             \
    }                                                                                                         \
    return ST_OK;                                                                                             \
  }

DEFINE_ONESIDED(double, f64, sqrt, fabs, hypot, fma, fmax, frexp, ldexp, 0x1p500, 0x1p-500)
DEFINE_ONESIDED(float, f32, sqrtf, fabsf, hypotf, fmaf, fmaxf, frexpf, ldexpf, 0x1p60f, 0x1p-60f)

/* The spectral phase of the two one-sided branches on the Gram mh (n x n,
 * binary64): sigma (working-precision values) and V (binary32), sorted
 * descending, sign of each V column fixed by its first largest entry
 * (jacobi.cpp:143-167), tiny-sigma check (thinsvd.cpp:22-26).
 *   choice 1 GramCholSvd: R = chol(mh), fl32(R) with the cast checks,
 *            one-sided Jacobi in binary32, sigma = sigma(R);
 *   choice 2 OneSidedJacobiOnGram: one-sided Jacobi of mh in binary64,
 *            sigma = fl32(sqrt(sigma(M))). */
int port_onesided_spectral(int choice, const double* mh, int64_t n, double tol, int max_sweeps, int sem,
                           double* sigma, float* v, port_jacobi_stats* stats, port_error* err) {
  set_err(err, ST_OK, 0, 0.0);
  if (choice != 1 && choice != 2) return set_err(err, ST_INVALID, 0, 0.0);
  const int dev = sem == PORT_SEM_DEVICE;
  const size_t nn = (size_t)(n * n);
  double* raw = (double*)malloc(sizeof(double) * (size_t)n);
  double* vd = (double*)malloc(sizeof(double) * nn); /* V widened (exact) */
  int st = ST_OK;
  if (choice == 1) {
    double* r = (double*)malloc(sizeof(double) * nn);
    st = port_cholesky_f64(mh, n, r, err);
    float* x = (float*)malloc(sizeof(float) * nn);
    float* vf = (float*)malloc(sizeof(float) * nn);
    float* sg = (float*)malloc(sizeof(float) * (size_t)n);
    if (st == ST_OK)
      for (int64_t j = 0; j < n && st == ST_OK; ++j) /* cast (dense.cpp:163-176) */
        for (int64_t i = 0; i < n; ++i) {
          const double val = r[j * n + i];
          if (!isfinite(val)) {
            st = set_err(err, ST_INVALID, i + 1, val);
            break;
          }
          if (fabs(val) > (double)FLT_MAX) {
            st = set_err(err, ST_CAST_OVERFLOW, i + 1, val);
            break;
          }
          x[j * n + i] = (float)val;
        }
    if (st == ST_OK) {
      const double t = tol > 0.0 ? tol : (double)n * 0x1p-24;
      st = onesided_f32(x, vf, n, n, t, max_sweeps, dev, sg, stats, err);
    }
    if (st == ST_OK) {
      for (int64_t j = 0; j < n; ++j) raw[j] = (double)sg[j];
      for (size_t k = 0; k < nn; ++k) vd[k] = (double)vf[k];
    }
    free(r);
    free(x);
    free(vf);
    free(sg);
  } else {
    double* x = (double*)malloc(sizeof(double) * nn);
    memcpy(x, mh, sizeof(double) * nn);
    const double t = tol > 0.0 ? tol : (double)n * 0x1p-53;
    st = onesided_f64(x, vd, n, n, t, max_sweeps, dev, raw, stats, err);
    free(x);
  }
  if (st == ST_OK) {
    for (int64_t j = 0; j < n; ++j)
      if (!(raw[j] > 0.0)) { /* jacobi.cpp:113-114 */
        st = set_err(err, ST_ZERO_COLUMN, j + 1, 0.0);
        break;
      }
  }
  if (st == ST_OK) {
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    descending_perm_f64(raw, n, perm);
    for (int64_t jj = 0; jj < n; ++jj) {
      const int64_t src = perm[jj];
      const double* vc = vd + src * n;
      int64_t imax = 0;
      double amax = -1.0;
      for (int64_t i = 0; i < n; ++i)
        if (fabs(vc[i]) > amax) {
          amax = fabs(vc[i]);
          imax = i;
        }
      const int flip = vc[imax] < 0.0;
      for (int64_t i = 0; i < n; ++i) v[jj * n + i] = (float)(flip ? -vc[i] : vc[i]);
      sigma[jj] = choice == 1 ? raw[src] : (double)(float)sqrt(raw[src]);
    }
    free(perm);
    for (int64_t i = 0; i < n; ++i) /* check_sigma_normal */
      if ((float)sigma[i] < FLT_MIN) {
        st = set_err(err, ST_TINY_SV, i + 1, sigma[i]);
        break;
      }
  }
  free(raw);
  free(vd);
  return st;
}

/* Row-wise forward substitution Q(i,:) R = A(i,:) in binary32
 * (thinsvd.cpp:136-152): per entry, subtract q_k r_kj for k ascending
 * (product and difference rounded separately), then divide. Device K10
 * performs the same sequence. */
void port_cholqr_solve(const float* a, int64_t m, int64_t n, const float* r, float* q) {
  for (int64_t j = 0; j < n; ++j) {
    float* qj = q + j * m;
    const float* aj = a + j * m;
    for (int64_t i = 0; i < m; ++i) qj[i] = aj[i];
    for (int64_t k = 0; k < j; ++k) {
      const float rkj = r[j * n + k];
      const float* qk = q + k * m;
      for (int64_t i = 0; i < m; ++i) qj[i] -= qk[i] * rkj;
    }
    const float rjj = r[j * n + j];
    for (int64_t i = 0; i < m; ++i) qj[i] /= rjj;
  }
}

/* mp_cholesky_qr (thinsvd.cpp:125-154) with the reference's own Gram
 * (gram_impl, dense.cpp:15-36: one accumulator per entry, ascending rows). */
int port_cholesky_qr_f32(const float* a, int64_t m, int64_t n, float* q, float* r, port_error* err) {
  set_err(err, ST_OK, 0, 0.0);
  if (m < n || n < 1) return set_err(err, ST_INVALID, 0, 0.0);
  const size_t nn = (size_t)(n * n);
  double* g = (double*)calloc(nn, sizeof(double));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i <= j; ++i) {
      double acc = 0.0;
      const float* ci = a + i * m;
      const float* cj = a + j * m;
      for (int64_t k = 0; k < m; ++k) acc += (double)ci[k] * (double)cj[k];
      g[j * n + i] = acc;
      g[i * n + j] = acc;
    }
  double* rh = (double*)malloc(sizeof(double) * nn);
  int st = port_cholesky_f64(g, n, rh, err);
  if (st == ST_OK)
    for (int64_t j = 0; j < n && st == ST_OK; ++j)
      for (int64_t i = 0; i < n; ++i) {
        const double v = rh[j * n + i];
        if (!isfinite(v)) {
          st = set_err(err, ST_INVALID, i + 1, v);
          break;
        }
        if (fabs(v) > (double)FLT_MAX) {
          st = set_err(err, ST_CAST_OVERFLOW, i + 1, v);
          break;
        }
        r[j * n + i] = (float)v;
      }
  if (st == ST_OK) port_cholqr_solve(a, m, n, r, q);
  free(g);
  free(rh);
  return st;
}

/* ======================================================================== */
/* fp32 thin SVD (proj/src/thinsvd.cpp:49-123)                              */
/* ======================================================================== */

typedef struct {
  const float* a;
  const float* w;
  float* u;
  int64_t m, n, j0, j1;
  int fma_chain;
} av_job;

/* matmul_impl (dense.cpp:83-96), jli order, f32; device semantics use one
 * fmaf chain per output entry over ascending l (same order). */
static void* av_worker(void* arg) {
  av_job* j = (av_job*)arg;
  const int64_t m = j->m, n = j->n;
  for (int64_t c = j->j0; c < j->j1; ++c) {
    float* uc = j->u + c * m;
    for (int64_t i = 0; i < m; ++i) uc[i] = 0.0f;
    for (int64_t l = 0; l < n; ++l) {
      const float blj = j->w[c * n + l];
      const float* al = j->a + l * m;
      if (j->fma_chain)
        for (int64_t i = 0; i < m; ++i) uc[i] = fmaf(al[i], blj, uc[i]);
      else
        for (int64_t i = 0; i < m; ++i) uc[i] += al[i] * blj;
    }
  }
  return NULL;
}

/* U = A W alone (w: n x n column-major), device semantics (fmaf chain). */
int port_av_f32(const float* a, int64_t m, int64_t n, const float* w, float* u, int threads) {
  int nt = threads < (int)n ? threads : (int)n;
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  pthread_t th[64];
  av_job jobs[64];
  for (int t = 0; t < nt; ++t) {
    jobs[t] = (av_job){a, w, u, m, n, n * t / nt, n * (t + 1) / nt, 1};
    pthread_create(&th[t], NULL, av_worker, &jobs[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  return ST_OK;
}

int port_thin_svd_f32(const float* a, int64_t m, int64_t n, int threads, int sem,
                      float* u, double* sigma, float* v, double* times5,
                      port_error* err) {
  return port_thin_svd_f32_choice(a, m, n, threads, sem, 0, u, sigma, v, times5, err);
}

int port_thin_svd_f32_choice(const float* a, int64_t m, int64_t n, int threads, int sem, int choice,
                             float* u, double* sigma, float* v, double* times5, port_error* err) {
  const double t0 = now_s();
  set_err(err, ST_OK, 0, 0.0);
  if (m < n || n < 1) return set_err(err, ST_INVALID, 0, 0.0);
  if (threads < 1) return set_err(err, ST_INVALID, 0, 0.0);
  const int64_t blocks = m < 16 ? m : 16; /* thinsvd.cpp:66 */
  double* mh = (double*)malloc(sizeof(double) * (size_t)(n * n));
  const double tg = now_s();
  int st = port_partitioned_gram_f32(a, m, n, blocks, mh);
  const double t_gram = now_s() - tg;
  if (st != ST_OK) {
    free(mh);
    return set_err(err, st, 0, 0.0);
  }
  const double te = now_s();
  if (choice != 0) {
    st = port_onesided_spectral(choice, mh, n, 0.0, 30, sem, sigma, v, NULL, err);
    free(mh);
    if (st != ST_OK) return st;
  } else {
    double* lam = (double*)malloc(sizeof(double) * (size_t)n);
    double* vh = (double*)malloc(sizeof(double) * (size_t)(n * n));
    st = port_twosided_jacobi_f64(mh, n, 0.0, 30, sem, lam, vh, NULL, err);
    free(mh);
    if (st != ST_OK) {
      free(lam);
      free(vh);
      return st;
    }
    for (int64_t i = 0; i < n; ++i) sigma[i] = (double)(float)sqrt(lam[i]);
    for (int64_t k = 0; k < n * n; ++k) v[k] = (float)vh[k];
    free(lam);
    free(vh);
  }
  for (int64_t i = 0; i < n; ++i) /* check_sigma_normal, thinsvd.cpp:22-26 */
    if ((float)sigma[i] < FLT_MIN) return set_err(err, ST_TINY_SV, i + 1, sigma[i]);
  const double t_eig = now_s() - te;
  const double tu = now_s();
  /* scale_columns(v, sigma, invert) (dense.cpp:220-232): true f32 division */
  float* w = (float*)malloc(sizeof(float) * (size_t)(n * n));
  for (int64_t j = 0; j < n; ++j) {
    const float sj = (float)sigma[j];
    if (sj == 0.0f) {
      free(w);
      return set_err(err, ST_ZERO_DIVISOR, j + 1, 0.0);
    }
    for (int64_t i = 0; i < n; ++i) w[j * n + i] = v[j * n + i] / sj;
  }
  /* the reference's matmul is single-threaded; threading over output
   * columns does not change any bit (each entry's order is fixed). */
  int nt = threads < (int)n ? threads : (int)n;
  if (nt > 64) nt = 64;
  pthread_t th[64];
  av_job jobs[64];
  for (int t = 0; t < nt; ++t) {
    jobs[t] = (av_job){a, w, u, m, n, n * t / nt, n * (t + 1) / nt, sem == PORT_SEM_DEVICE};
    pthread_create(&th[t], NULL, av_worker, &jobs[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  free(w);
  const double t_u = now_s() - tu;
  if (times5) {
    times5[0] = t_gram;
    times5[1] = t_eig;
    times5[2] = t_u;
    times5[4] = now_s() - t0;
    times5[3] = times5[4] - t_gram - t_eig - t_u;
  }
  return ST_OK;
}

/* ======================================================================== */
/* Double-double (proj/tests/support/dd.cpp:10-65)                          */
/* ======================================================================== */

typedef struct {
  double hi, lo;
} dd;

static inline dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return (dd){s, e};
}
static inline dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return (dd){s, b - (s - a)};
}
static inline dd two_prod(double a, double b) {
  const double p = a * b;
  return (dd){p, fma(a, b, -p)};
}
static inline dd dd_from(double x) { return (dd){x, 0.0}; }
static inline dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  s.lo += a.lo + b.lo;
  return quick_two_sum(s.hi, s.lo);
}
static inline dd dd_neg(dd a) { return (dd){-a.hi, -a.lo}; }
static inline dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
static inline dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
static inline dd dd_div(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  dd r = dd_sub(a, dd_mul(dd_from(q1), b));
  const double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul(dd_from(q2), b));
  const double q3 = r.hi / b.hi;
  return dd_add(quick_two_sum(q1, q2), dd_from(q3));
}
static inline dd dd_sqrt(dd a) {
  if (a.hi == 0.0 && a.lo == 0.0) return (dd){0.0, 0.0};
  const double s = sqrt(a.hi);
  const dd e = dd_sub(a, two_prod(s, s));
  const double corr = e.hi / (2.0 * s);
  return quick_two_sum(s, corr);
}
static inline dd dd_abs(dd a) { return a.hi < 0.0 ? dd_neg(a) : a; }
static inline int dd_le(dd a, dd b) { return a.hi < b.hi || (a.hi == b.hi && a.lo <= b.lo); }
static inline int dd_gt0(dd a) { return a.hi > 0.0 || (a.hi == 0.0 && a.lo > 0.0); }
static inline dd dd_scale2(dd a) { return (dd){2.0 * a.hi, 2.0 * a.lo}; }
/* sqrt(1 + z^2) in double-double; z^2 stays finite below 2^500. */
static inline dd dd_hyp1(dd z) {
  const dd az = dd_abs(z);
  if (az.hi >= 0x1p500) return az;
  return dd_sqrt(dd_add(dd_mul(z, z), dd_from(1.0)));
}

void port_dd_add(double ah, double al, double bh, double bl, double* rh, double* rl) {
  dd r = dd_add((dd){ah, al}, (dd){bh, bl});
  *rh = r.hi;
  *rl = r.lo;
}
void port_dd_mul(double ah, double al, double bh, double bl, double* rh, double* rl) {
  dd r = dd_mul((dd){ah, al}, (dd){bh, bl});
  *rh = r.hi;
  *rl = r.lo;
}
void port_dd_div(double ah, double al, double bh, double bl, double* rh, double* rl) {
  dd r = dd_div((dd){ah, al}, (dd){bh, bl});
  *rh = r.hi;
  *rl = r.lo;
}
void port_dd_sqrt(double ah, double al, double* rh, double* rl) {
  dd r = dd_sqrt((dd){ah, al});
  *rh = r.hi;
  *rl = r.lo;
}

/* dd_gram (dd.cpp:75-88): acc = dd_add(acc, two_prod(a_ki, a_kj)), k
 * ascending, upper triangle mirrored. Threads split the columns j. */
typedef struct {
  const double* a;
  int64_t m, n;
  int tid, nt;
  double *hi, *lo;
} ddg_job;

static void* ddg_worker(void* arg) {
  ddg_job* J = (ddg_job*)arg;
  const int64_t m = J->m, n = J->n;
  /* interleave columns so threads get balanced triangles */
  for (int64_t j = J->tid; j < n; j += J->nt) {
    const double* cj = J->a + j * m;
    for (int64_t i = 0; i <= j; ++i) {
      const double* ci = J->a + i * m;
      dd acc = {0.0, 0.0};
      for (int64_t k = 0; k < m; ++k) acc = dd_add(acc, two_prod(ci[k], cj[k]));
      J->hi[j * n + i] = acc.hi;
      J->lo[j * n + i] = acc.lo;
      J->hi[i * n + j] = acc.hi;
      J->lo[i * n + j] = acc.lo;
    }
  }
  return NULL;
}

int port_dd_gram(const double* a, int64_t m, int64_t n, int threads, double* hi,
                 double* lo) {
  if (m < 1 || n < 1) return ST_INVALID;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  ddg_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (ddg_job){a, m, n, t, threads, hi, lo};
    pthread_create(&th[t], NULL, ddg_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  return ST_OK;
}

/* K2z, the double-double Gram on the int8 tensor cores
 * (paper_2603_11953_b200/csrc/gram_ozaki.cu), replayed bit for bit: the
 * per-split column exponents, the 11 balanced 8-bit digits of
 * trunc(x 2^(86 - E)), the exact integer digit-product sums per weight and
 * exact-accumulation span, their conversion to double-double
 * (V = sum_k acc_k 2^(8k), acc_k of weight w_hi - k; (fl(V), V - fl(V))
 * scaled by 2^(E_i + E_j + 4 - 8 w_hi)), the running dd_add per partial
 * slot (split * 6 + sub-group), then the engine's combine: slots of a logical block
 * summed in order from zero, blocks along the reference tree
 * (parallel_gram.cpp:93-102). Semantics follow dd_gram (dd.cpp:75-88) up to
 * the digit truncation. */
#define OZ_L 11
#define OZ_G 6
/* sub-group i: weight quad (w_hi, nw weights w_hi - k) and steps [pa, pb]
 * (gram_ozaki.cu sub_group) */
static void oz_sub_group(int i, int* whi, int* nw, int* pa, int* pb) {
  for (int q = 0; q < 3; ++q) {
    const int h = 12 - 4 * q, d = h - 1, parts = (d + 3) / 4;
    if (i < parts) {
      const int base = d / parts, extra = d % parts;
      *pa = 1 + i * base + (i < extra ? i : extra);
      *pb = *pa + base + (i < extra ? 1 : 0) - 1;
      *whi = h;
      *nw = q == 2 ? 3 : 4;
      return;
    }
    i -= parts;
  }
  *whi = *nw = *pa = *pb = 0;
}
#define OZ_BAD (1 << 20)
static void oz_fixed88(double x, int e_col, uint32_t w[3]) {
  uint64_t bits;
  memcpy(&bits, &x, 8);
  const int e = (int)((bits >> 52) & 0x7ff);
  const uint64_t mant = (bits & 0xFFFFFFFFFFFFFull) | (e ? (1ull << 52) : 0ull);
  const int s = (e ? e : 1) - 989 - e_col;
  uint64_t lo = 0, hi = 0;
  if (s >= 0) {
    lo = mant << s;
    hi = s ? (mant >> (64 - s)) : 0ull;
  } else if (s > -64) {
    lo = mant >> (-s);
  }
  const uint64_t olo = 0x8080808080808080ull, ohi = 0x808080ull;
  uint64_t rlo, rhi;
  if ((int64_t)bits >= 0) {
    rlo = olo + lo;
    rhi = ohi + hi + (rlo < lo ? 1ull : 0ull);
  } else {
    rlo = olo - lo;
    rhi = ohi - hi - (olo < lo ? 1ull : 0ull);
  }
  w[0] = (uint32_t)rlo;
  w[1] = (uint32_t)(rlo >> 32);
  w[2] = (uint32_t)rhi;
}

void port_oz_sub_group(int i, int* whi, int* nw, int* pa, int* pb) { oz_sub_group(i, whi, nw, pa, pb); }

int port_gram_dd_ozaki(const double* a, int64_t m, int64_t n, int nsplit, const int* scb, int nblocks,
                       const int* bsb, int span_cap, double* out_hi, double* out_lo) {
  if (m < 1 || n < 1 || nsplit < 1 || nblocks < 1 || nblocks > 16) return ST_INVALID;
  // the schedule must be a K2z chunk schedule covering every row exactly once
  if (scb[0] != 0 || (int64_t)scb[nsplit] * 32 < m || bsb[0] != 0 || bsb[nblocks] != nsplit) return ST_INVALID;
  for (int s = 0; s < nsplit; ++s)
    if (scb[s + 1] < scb[s]) return ST_INVALID;
  for (int b = 0; b < nblocks; ++b)
    if (bsb[b + 1] < bsb[b]) return ST_INVALID;
  int* E = (int*)malloc(sizeof(int) * (size_t)(nsplit * n));
  for (int s = 0; s < nsplit; ++s) {
    const int64_t r0 = (int64_t)scb[s] * 32;
    int64_t r1 = (int64_t)scb[s + 1] * 32;
    if (r1 > m) r1 = m;
    for (int64_t c = 0; c < n; ++c) {
      double mx = 0.0;
      int bad = 0;
      for (int64_t r = r0; r < r1; ++r) {
        const double v = fabs(a[c * m + r]);
        if (!(v <= DBL_MAX)) bad = 1;
        mx = fmax(mx, v);
      }
      int e = 0;
      if (mx > 0.0) frexp(mx, &e);
      E[s * n + c] = bad ? OZ_BAD : e;
    }
  }
  int8_t* D = (int8_t*)malloc((size_t)(m * n * OZ_L));
  int* rsplit = (int*)malloc(sizeof(int) * (size_t)m);
  for (int s = 0; s < nsplit; ++s)
    for (int64_t r = (int64_t)scb[s] * 32; r < (int64_t)scb[s + 1] * 32 && r < m; ++r) rsplit[r] = s;
  for (int64_t r = 0; r < m; ++r)
    for (int64_t c = 0; c < n; ++c) {
      const int e = E[rsplit[r] * n + c];
      uint32_t w[3];
      oz_fixed88(e == OZ_BAD ? 0.0 : a[c * m + r], e, w);
      for (int p = 1; p <= OZ_L; ++p) {
        const int b = OZ_L - p;
        D[(r * n + c) * OZ_L + p - 1] = (int8_t)(((w[b >> 2] >> (8 * (b & 3))) & 0xffu) ^ 0x80u);
      }
    }
  const int64_t nslot = (int64_t)nsplit * OZ_G;
  dd* part = (dd*)calloc((size_t)(nslot * n * n), sizeof(dd));
  for (int s = 0; s < nsplit; ++s)
    for (int g = 0; g < OZ_G; ++g) {
      int whi, nw, pa, pb;
      oz_sub_group(g, &whi, &nw, &pa, &pb);
      const int maxpairs = pb - pa + 1;
      int span = 1;
      while (span * 2 * maxpairs < 4096) span *= 2;
      if (span > span_cap) span = span_cap;
      const int64_t c0 = scb[s], c1 = scb[s + 1];
      dd* P = part + ((int64_t)s * OZ_G + g) * n * n;
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i; j < n; ++j) {
          dd run = {0.0, 0.0};
          const int ei = E[s * n + i], ej = E[s * n + j];
          for (int64_t ch = c0; ch < c1; ch += span) {
            const int64_t ce = ch + span < c1 ? ch + span : c1;
            int64_t acc[4] = {0, 0, 0, 0};
            for (int64_t r = ch * 32; r < ce * 32 && r < m; ++r) {
              const int8_t* di = D + (r * n + i) * OZ_L - 1; /* di[p], p = 1..11 */
              const int8_t* dj = D + (r * n + j) * OZ_L - 1;
              for (int p = pa; p <= pb; ++p)
                for (int k = 0; k < nw; ++k)
                  if (p - k >= 1) acc[k] += (int64_t)di[p - k] * dj[whi - p]; /* W_k: (p - k, w_hi - p) */
            }
            const int64_t v = acc[0] + acc[1] * 256 + acc[2] * 65536 + acc[3] * 16777216;
            const double h = (double)v;
            const double l = (double)(v - (int64_t)h);
            dd t;
            if (ei == OZ_BAD || ej == OZ_BAD) {
              t.hi = NAN;
              t.lo = 0.0;
            } else {
              const int sc = ei + ej + 4 - 8 * whi;
              t.hi = scalbn(h, sc);
              t.lo = scalbn(l, sc);
            }
            run = ch == c0 ? t : dd_add(run, t);
          }
          P[i * n + j] = run;
        }
    }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j) {
      dd slot[16];
      for (int b = 0; b < nblocks; ++b) {
        dd acc = {0.0, 0.0};
        for (int64_t k = (int64_t)bsb[b] * OZ_G; k < (int64_t)bsb[b + 1] * OZ_G; ++k) acc = dd_add(acc, part[k * n * n + i * n + j]);
        slot[b] = acc;
      }
      for (int width = 1; width < nblocks; width *= 2)
        for (int b = 0; b + width < nblocks; b += 2 * width) slot[b] = dd_add(slot[b], slot[b + width]);
      out_hi[j * n + i] = out_hi[i * n + j] = slot[0].hi;
      out_lo[j * n + i] = out_lo[i * n + j] = slot[0].lo;
    }
  free(part);
  free(D);
  free(rsplit);
  free(E);
  return ST_OK;
}

static void finish_dd(const dd* A, const dd* V, int64_t n, double* lam_hi, double* lam_lo,
                      double* vhi, double* vlo) {
  /* sort keys: dd values compared lexicographically (hi, lo); stable. */
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  for (int64_t i = 1; i < n; ++i) {
    const int64_t x = perm[i];
    const dd kx = A[x * n + x];
    int64_t j = i - 1;
    while (j >= 0) {
      const dd kj = A[perm[j] * n + perm[j]];
      if (!(kx.hi > kj.hi || (kx.hi == kj.hi && kx.lo > kj.lo))) break;
      perm[j + 1] = perm[j];
      --j;
    }
    perm[j + 1] = x;
  }
  for (int64_t jj = 0; jj < n; ++jj) {
    const int64_t src = perm[jj];
    const dd* vc = V + src * n;
    int64_t imax = 0;
    dd amax = {-1.0, 0.0};
    for (int64_t i = 0; i < n; ++i) {
      const dd av = dd_abs(vc[i]);
      if (av.hi > amax.hi || (av.hi == amax.hi && av.lo > amax.lo)) {
        amax = av;
        imax = i;
      }
    }
    const int flip = vc[imax].hi < 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const dd x = flip ? dd_neg(vc[i]) : vc[i];
      vhi[jj * n + i] = x.hi;
      vlo[jj * n + i] = x.lo;
    }
    lam_hi[jj] = A[src * n + src].hi;
    lam_lo[jj] = A[src * n + src].lo;
  }
  free(perm);
}

typedef struct {
  dd c, s, t;
  int act;
} dd_rot;

/* One rotation from the 2x2 diagonal block, jacobi.cpp:211-224 in dd. */
static int dd_make_rotation(dd aii, dd ajj, dd aij, dd tol, double* worst, dd_rot* r) {
  const dd thresh = dd_mul(dd_mul(tol, dd_sqrt(aii)), dd_sqrt(ajj));
  const double ratio = fabs(aij.hi) / sqrt(aii.hi * ajj.hi);
  if (*worst < ratio) *worst = ratio;
  r->act = 0;
  r->c = dd_from(1.0);
  r->s = dd_from(0.0);
  r->t = dd_from(0.0);
  if (dd_le(dd_abs(aij), thresh)) return 0;
  const dd zeta = dd_div(dd_sub(ajj, aii), dd_scale2(aij));
  const dd t = dd_div(dd_from(zeta.hi >= 0.0 ? 1.0 : -1.0), dd_add(dd_abs(zeta), dd_hyp1(zeta)));
  const dd c = dd_div(dd_from(1.0), dd_hyp1(t));
  r->c = c;
  r->s = dd_mul(c, t);
  r->t = t;
  r->act = 1;
  return 1;
}

/* Device formula (jacobi.cu Arith<double2>::rotation). */
static int dd_make_rotation_dev(dd aii, dd ajj, dd aij, double tol, double* worst, int want_ratio,
                                dd_rot* r) {
  const double pr = aii.hi * ajj.hi;
  const double thresh = (pr > 0x1p-1000 && pr < 0x1p1000) ? tol * sqrt(pr) : tol * sqrt(aii.hi) * sqrt(ajj.hi);
  if (want_ratio) {
    const double ratio = fabs(aij.hi) / sqrt(pr);
    if (*worst < ratio) *worst = ratio;
  }
  r->act = 0;
  r->c = dd_from(1.0);
  r->s = dd_from(0.0);
  r->t = dd_from(0.0);
  if (fabs(aij.hi) <= thresh) return 0;
  dd x = dd_sub(ajj, aii), y = dd_scale2(aij);
  const int xzero = x.hi == 0.0, xpos = x.hi > 0.0;
  const double big = fmax(fabs(x.hi), fabs(y.hi));
  if (!(big < 0x1p250 && big > 0x1p-250)) {
    int e;
    frexp(big, &e);
    x = (dd){ldexp(x.hi, -e), ldexp(x.lo, -e)};
    y = (dd){ldexp(y.hi, -e), ldexp(y.lo, -e)};
  }
  const dd ax = dd_abs(x);
  const dd q = dd_add(dd_mul(x, x), dd_mul(y, y));
  const double r0 = sqrt(q.hi), iq = 1.0 / q.hi;
  const double ir = r0 * iq;
  const double id = 1.0 / (ax.hi + r0);
  const dd er = dd_sub(q, two_prod(r0, r0));
  const dd rr = quick_two_sum(r0, er.hi * (0.5 * ir));
  const dd den = dd_add(ax, rr);
  dd t = dd_from(1.0);
  if (!xzero) {
    const dd ys = xpos ? y : dd_neg(y);
    const double t0 = ys.hi * id;
    const dd et = dd_sub(ys, dd_mul(dd_from(t0), den));
    t = quick_two_sum(t0, et.hi * id);
  }
  const double u0 = ax.hi * ir;
  const dd eu = dd_sub(ax, dd_mul(dd_from(u0), rr));
  const dd u = quick_two_sum(u0, eu.hi * ir);
  const dd c2 = dd_add(dd_from(0.5), (dd){0.5 * u.hi, 0.5 * u.lo});
  const double c0 = sqrt(c2.hi), ic2 = 1.0 / c2.hi;
  const dd ec = dd_sub(c2, two_prod(c0, c0));
  const dd c = quick_two_sum(c0, ec.hi * (0.5 * (c0 * ic2)));
  r->c = c;
  r->s = dd_mul(c, t);
  r->t = t;
  r->act = 1;
  return 1;
}


static inline dd ddrot_lo(dd c, dd s, dd x, dd y) { return dd_sub(dd_mul(c, x), dd_mul(s, y)); }
static inline dd ddrot_hi(dd c, dd s, dd x, dd y) { return dd_add(dd_mul(s, x), dd_mul(c, y)); }

static int jacobi_cyclic_dd(dd* A, dd* V, int64_t n, dd tol, int max_sweeps,
                            port_jacobi_stats* st, port_error* err) {
#define AE(i, j) A[(j) * n + (i)]
  double worst = 0.0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    worst = 0.0;
    for (int64_t i = 0; i < n - 1; ++i)
      for (int64_t j = i + 1; j < n; ++j) {
        const dd aii = AE(i, i), ajj = AE(j, j), aij = AE(i, j);
        dd_rot r;
        if (!dd_make_rotation(aii, ajj, aij, tol, &worst, &r)) continue;
        for (int64_t k = 0; k < n; ++k) {
          if (k == i || k == j) continue;
          const dd aki = AE(k, i), akj = AE(k, j);
          const dd ni = ddrot_lo(r.c, r.s, aki, akj), nj = ddrot_hi(r.c, r.s, aki, akj);
          AE(k, i) = ni;
          AE(i, k) = ni;
          AE(k, j) = nj;
          AE(j, k) = nj;
        }
        AE(i, i) = dd_sub(aii, dd_mul(r.t, aij));
        AE(j, j) = dd_add(ajj, dd_mul(r.t, aij));
        AE(i, j) = dd_from(0.0);
        AE(j, i) = dd_from(0.0);
        if (!dd_gt0(AE(i, i))) return set_err(err, ST_NPD, i + 1, AE(i, i).hi);
        if (!dd_gt0(AE(j, j))) return set_err(err, ST_NPD, j + 1, AE(j, j).hi);
        dd* vi = V + i * n;
        dd* vj = V + j * n;
        for (int64_t k = 0; k < n; ++k) {
          const dd t1 = vi[k], t2 = vj[k];
          vi[k] = ddrot_lo(r.c, r.s, t1, t2);
          vj[k] = ddrot_hi(r.c, r.s, t1, t2);
        }
        rotated = 1;
        if (st) ++st->rotations;
      }
    if (st) ++st->sweeps;
    if (!rotated) return ST_OK;
  }
  return set_err(err, ST_NOCONV, max_sweeps, worst);
#undef AE
}

static int jacobi_rr_dd(dd* A, dd* V, int64_t n, dd tol, int max_sweeps,
                        port_jacobi_stats* st, port_error* err) {
#define AE(i, j) A[(j) * n + (i)]
  const int64_t N = n + (n & 1), np = N / 2;
  int64_t* P = (int64_t*)malloc(sizeof(int64_t) * (size_t)np);
  int64_t* Q = (int64_t*)malloc(sizeof(int64_t) * (size_t)np);
  dd_rot* R = (dd_rot*)malloc(sizeof(dd_rot) * (size_t)np);
  double worst = 0.0;
  int status = ST_NOCONV;
  for (int sweep = 0; sweep < max_sweeps && status == ST_NOCONV; ++sweep) {
    int64_t rot_in_sweep = 0;
    worst = 0.0;
    for (int64_t r = 0; r < N - 1; ++r) {
      for (int64_t k = 0; k < np; ++k) {
        port_rr_pair(n, r, k, &P[k], &Q[k]);
        R[k].act = 0;
        if (Q[k] >= n) continue;
        rot_in_sweep += dd_make_rotation_dev(AE(P[k], P[k]), AE(Q[k], Q[k]), AE(P[k], Q[k]), tol.hi,
                                             &worst, sweep + 1 == max_sweeps, &R[k]);
      }
      for (int64_t a = 0; a < np; ++a)
        for (int64_t b = a + 1; b < np; ++b) {
          if (!R[a].act && !R[b].act) continue;
          const int64_t rows[2] = {P[a], Q[a]}, cols[2] = {P[b], Q[b]};
          const int nr = Q[a] < n ? 2 : 1, nc = Q[b] < n ? 2 : 1;
          dd x[2][2] = {{{0, 0}, {0, 0}}, {{0, 0}, {0, 0}}};
          for (int u = 0; u < nr; ++u)
            for (int w = 0; w < nc; ++w) x[u][w] = AE(rows[u], cols[w]);
          if (R[b].act)
            for (int u = 0; u < nr; ++u) {
              const dd x0 = x[u][0], x1 = x[u][1];
              x[u][0] = ddrot_lo(R[b].c, R[b].s, x0, x1);
              x[u][1] = ddrot_hi(R[b].c, R[b].s, x0, x1);
            }
          if (R[a].act)
            for (int w = 0; w < nc; ++w) {
              const dd y0 = x[0][w], y1 = x[1][w];
              x[0][w] = ddrot_lo(R[a].c, R[a].s, y0, y1);
              x[1][w] = ddrot_hi(R[a].c, R[a].s, y0, y1);
            }
          for (int u = 0; u < nr; ++u)
            for (int w = 0; w < nc; ++w) {
              AE(rows[u], cols[w]) = x[u][w];
              AE(cols[w], rows[u]) = x[u][w];
            }
        }
      int64_t bad_idx = 0;
      double bad_val = 0.0;
      for (int64_t k = 0; k < np; ++k) {
        if (!R[k].act) continue;
        const int64_t p = P[k], q = Q[k];
        const dd tapq = dd_mul(R[k].t, AE(p, q));
        const dd app = dd_sub(AE(p, p), tapq);
        const dd aqq = dd_add(AE(q, q), tapq);
        AE(p, p) = app;
        AE(q, q) = aqq;
        AE(p, q) = dd_from(0.0);
        AE(q, p) = dd_from(0.0);
        if (!dd_gt0(app) && (bad_idx == 0 || p + 1 < bad_idx)) {
          bad_idx = p + 1;
          bad_val = app.hi;
        }
        if (!dd_gt0(aqq) && (bad_idx == 0 || q + 1 < bad_idx)) {
          bad_idx = q + 1;
          bad_val = aqq.hi;
        }
      }
      if (bad_idx) {
        status = set_err(err, ST_NPD, bad_idx, bad_val);
        break;
      }
      for (int64_t k = 0; k < np; ++k) {
        if (!R[k].act) continue;
        dd* vp = V + P[k] * n;
        dd* vq = V + Q[k] * n;
        for (int64_t x = 0; x < n; ++x) {
          const dd t1 = vp[x], t2 = vq[x];
          vp[x] = ddrot_lo(R[k].c, R[k].s, t1, t2);
          vq[x] = ddrot_hi(R[k].c, R[k].s, t1, t2);
        }
      }
    }
    if (status != ST_NOCONV) break;
    if (st) {
      ++st->sweeps;
      st->rotations += rot_in_sweep;
    }
    if (rot_in_sweep == 0) status = ST_OK;
  }
  if (status == ST_NOCONV) set_err(err, ST_NOCONV, max_sweeps, worst);
  free(P);
  free(Q);
  free(R);
  return status;
#undef AE
}

int port_twosided_jacobi_dd(const double* mhi, const double* mlo, int64_t n, double tol,
                            int max_sweeps, int sem, double* lam_hi, double* lam_lo,
                            double* vhi, double* vlo, port_jacobi_stats* stats,
                            port_error* err) {
  set_err(err, ST_OK, 0, 0.0);
  if (n < 1 || max_sweeps < 1) return set_err(err, ST_INVALID, 0, 0.0);
  if (!(tol > 0.0)) tol = (double)n * 0x1p-104; /* u_dd = 2^-104 */
  if (stats) {
    stats->sweeps = 0;
    stats->rotations = 0;
    stats->pairs_per_sweep = n * (n - 1) / 2;
  }
  dd* A = (dd*)malloc(sizeof(dd) * (size_t)(n * n));
  dd* V = (dd*)calloc((size_t)(n * n), sizeof(dd));
  for (int64_t k = 0; k < n * n; ++k) A[k] = (dd){mhi[k], mlo ? mlo[k] : 0.0};
  for (int64_t i = 0; i < n; ++i) V[i * n + i] = dd_from(1.0);
  int st = ST_OK;
  for (int64_t k = 0; k < n; ++k)
    if (!dd_gt0(A[k * n + k])) {
      st = set_err(err, ST_NPD, k + 1, A[k * n + k].hi);
      break;
    }
  if (st == ST_OK)
    st = sem == PORT_SEM_REFERENCE ? jacobi_cyclic_dd(A, V, n, dd_from(tol), max_sweeps, stats, err)
                                   : jacobi_rr_dd(A, V, n, dd_from(tol), max_sweeps, stats, err);
  if (st == ST_OK) finish_dd(A, V, n, lam_hi, lam_lo, vhi, vlo);
  free(A);
  free(V);
  return st;
}

typedef struct {
  const double* a;
  const double* w;
  double* u;
  int64_t m, n, j0, j1;
} av64_job;

/* U = A*W in fp64, one fma chain per entry over ascending l. */
static void* av64_worker(void* arg) {
  av64_job* j = (av64_job*)arg;
  const int64_t m = j->m, n = j->n;
  for (int64_t c = j->j0; c < j->j1; ++c) {
    double* uc = j->u + c * m;
    for (int64_t i = 0; i < m; ++i) uc[i] = 0.0;
    for (int64_t l = 0; l < n; ++l) {
      const double blj = j->w[c * n + l];
      const double* al = j->a + l * m;
      for (int64_t i = 0; i < m; ++i) uc[i] = fma(al[i], blj, uc[i]);
    }
  }
  return NULL;
}

int port_thin_svd_f64dd(const double* a, int64_t m, int64_t n, int threads, int sem,
                        double* u, double* sigma, double* v, double* times5,
                        port_error* err) {
  const double t0 = now_s();
  set_err(err, ST_OK, 0, 0.0);
  if (m < n || n < 1 || threads < 1) return set_err(err, ST_INVALID, 0, 0.0);
  double* ghi = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* glo = (double*)malloc(sizeof(double) * (size_t)(n * n));
  const double tg = now_s();
  port_dd_gram(a, m, n, threads, ghi, glo);
  const double t_gram = now_s() - tg;
  const double te = now_s();
  double* lh = (double*)malloc(sizeof(double) * (size_t)n);
  double* ll = (double*)malloc(sizeof(double) * (size_t)n);
  double* vl = (double*)malloc(sizeof(double) * (size_t)(n * n));
  /* sweep cap of the double-double path: kDdMaxSweeps (include/mpsvd/thinsvd.hpp) */
  int st = port_twosided_jacobi_dd(ghi, glo, n, 0.0, 100, sem, lh, ll, v, vl, NULL, err);
  free(ghi);
  free(glo);
  free(vl);
  if (st != ST_OK) {
    free(lh);
    free(ll);
    return st;
  }
  for (int64_t i = 0; i < n; ++i) sigma[i] = dd_sqrt((dd){lh[i], ll[i]}).hi;
  free(lh);
  free(ll);
  for (int64_t i = 0; i < n; ++i)
    if (sigma[i] < DBL_MIN) return set_err(err, ST_TINY_SV, i + 1, sigma[i]);
  const double t_eig = now_s() - te;
  const double tu = now_s();
  double* w = (double*)malloc(sizeof(double) * (size_t)(n * n));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) w[j * n + i] = v[j * n + i] / sigma[j];
  int nt = threads < (int)n ? threads : (int)n;
  if (nt > 64) nt = 64;
  pthread_t th[64];
  av64_job jobs[64];
  for (int t = 0; t < nt; ++t) {
    jobs[t] = (av64_job){a, w, u, m, n, n * t / nt, n * (t + 1) / nt};
    pthread_create(&th[t], NULL, av64_worker, &jobs[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  free(w);
  const double t_u = now_s() - tu;
  if (times5) {
    times5[0] = t_gram;
    times5[1] = t_eig;
    times5[2] = t_u;
    times5[4] = now_s() - t0;
    times5[3] = times5[4] - t_gram - t_eig - t_u;
  }
  return ST_OK;
}

/* ======================================================================== */
/* orth_error (proj/src/dense.cpp:250-272), threaded over columns j         */
/* ======================================================================== */

typedef struct {
  const float* qf;
  const double* qd;
  int64_t m, n;
  int tid, nt;
  double sum;
} orth_job;

static void* orth_worker(void* arg) {
  orth_job* J = (orth_job*)arg;
  const int64_t m = J->m, n = J->n;
  double sum = 0.0;
  for (int64_t j = J->tid; j < n; j += J->nt)
    for (int64_t i = 0; i <= j; ++i) {
      double dot = 0.0;
      if (J->qf) {
        const float* ci = J->qf + i * m;
        const float* cj = J->qf + j * m;
        for (int64_t k = 0; k < m; ++k) dot += (double)ci[k] * (double)cj[k];
      } else {
        const double* ci = J->qd + i * m;
        const double* cj = J->qd + j * m;
        for (int64_t k = 0; k < m; ++k) dot += ci[k] * cj[k];
      }
      const double d = dot - (i == j ? 1.0 : 0.0);
      sum += (i == j) ? d * d : 2.0 * d * d;
    }
  J->sum = sum;
  return NULL;
}

static double orth_run(const float* qf, const double* qd, int64_t m, int64_t n, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  orth_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (orth_job){qf, qd, m, n, t, threads, 0.0};
    pthread_create(&th[t], NULL, orth_worker, &jobs[t]);
  }
  double sum = 0.0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    sum += jobs[t].sum;
  }
  return sqrt(sum);
}

double port_orth_error_f32(const float* q, int64_t m, int64_t n, int threads) {
  return orth_run(q, NULL, m, n, threads);
}
double port_orth_error_f64(const double* q, int64_t m, int64_t n, int threads) {
  return orth_run(NULL, q, m, n, threads);
}

/* ======================================================================== */
/* K1z restated (csrc/gram_ozaki32.cu): the binary64 Gram of a binary32 A   */
/* (n <= 128) by the int8 Ozaki scheme, bit for bit. Reference semantics:   */
/* partitioned_gram of cast(A, Higher) (proj/src/parallel_gram.cpp:79-112); */
/* this is the device's different exact-accumulation order, restated so the */
/* tests can pin the kernel bitwise; its accuracy against the reference is   */
/* checked separately (tests/test_ozaki32.py).                               */
/* ======================================================================== */

#define O32_ZERO_E (-160)
#define O32_HEAD 2

#define O32_C48 0x808080808080ull

static int o32_fexp_bits(uint32_t ab) {
  const int e8 = (int)(ab >> 23);
  if (e8) return e8 - 126;
  if (!ab) return -1000;
  return (32 - __builtin_clz(ab)) - 149;
}

static uint64_t o32_fixed48(uint32_t b, int E) {
  const uint32_t e8 = (b >> 23) & 0xFFu;
  if (e8 == 0xFFu) return O32_C48;
  const uint32_t mant = (b & 0x7FFFFFu) | (e8 ? 0x800000u : 0u);
  const int sh = (int)(e8 ? e8 : 1u) - 104 - E;
  uint64_t X = 0;
  if (mant) { /* round to nearest, ties to even */
    if (sh >= 0) {
      X = (uint64_t)mant << sh;
    } else if (sh > -64) {
      const int s = -sh;
      const uint64_t r = (uint64_t)mant >> s;
      const uint64_t rem = (uint64_t)mant - (r << s), half = 1ull << (s - 1);
      X = r + ((rem > half || (rem == half && (r & 1ull))) ? 1ull : 0ull);
    }
  }
  return (b >> 31) ? O32_C48 - X : O32_C48 + X;
}

static void o32_product(int g, int k, int* p, int* q, int* acc) {
  const int sh = 4 * k;
  *p = (int)(((g ? 0x322121u : 0x111321u) >> sh) & 15u);
  *q = (int)(((g ? 0x323445u : 0x123456u) >> sh) & 15u);
  *acc = (int)(((g ? 0x321100u : 0x321000u) >> sh) & 15u);
}

static dd o32_group_total(int g, int32_t a0, int32_t a1, int32_t a2, int32_t a3) {
  if (g == 0) {
    const int64_t vlo = (int64_t)a0 + (int64_t)a1 * 16777216LL;
    const int64_t vhi = (int64_t)a2 + (int64_t)a3 * 128LL;
    const double lh = (double)vlo;
    const double ll = (double)(vlo - (int64_t)lh);
    return dd_add((dd){(double)vhi * 4294967296.0, 0.0}, (dd){lh, ll});
  }
  const int64_t v = (int64_t)a0 * 2LL + (int64_t)a1 * 512LL + (int64_t)a2 * 65536LL + (int64_t)a3;
  return (dd){(double)v, 0.0};
}

typedef struct {
  const float* a;
  int64_t m, n, c0, c1;
  int g, accumulate, span_max;
  dd* P;      /* [128][128], [j][i] */
  int* bad;   /* [128] */
} O32Job;

static void* o32_worker(void* arg) {
  O32Job* J = (O32Job*)arg;
  const int64_t m = J->m, n = J->n;
  const int g = J->g;
  int64_t* acc = (int64_t*)calloc((size_t)4 * 128 * 128, sizeof(int64_t));
  int8_t* D = (int8_t*)malloc((size_t)6 * 64 * 128); /* [p][r][c], one 64-row step */
  int E[128];
  int64_t s8[128];
  for (int c = 0; c < 128; ++c) {
    E[c] = O32_ZERO_E;
    s8[c] = 0;
  }
  int span = -1, len = 0;
  const int base = g ? 47 : 40;
  /* the device pipeline moves 64-row steps (two chunks; a range with an
     odd chunk count ends on a half step whose second chunk is zero): span
     decisions are per step */
  uint32_t(*b)[128] = (uint32_t(*)[128])malloc(sizeof(uint32_t) * 64 * 128);
  for (int64_t ch = J->c0;; ch += 2) {
    const int end = ch >= J->c1;
    uint32_t mx[128];
    int fresh = 0;
    if (!end) {
      for (int c = 0; c < 128; ++c) {
        mx[c] = 0;
        for (int r = 0; r < 64; ++r) {
          const int64_t row = ch * 32 + r;
          uint32_t v = 0;
          if (ch + r / 32 < J->c1 && row < m && c < n) memcpy(&v, &J->a[c * m + row], 4);
          const uint32_t ab = v & 0x7FFFFFFFu;
          if (ab > mx[c]) mx[c] = ab; /* inf / NaN included: they force a new span */
          if ((ab >> 23) == 0xFFu) {  /* the column is flagged, the entry used as zero */
            J->bad[c] = 1;
            v = 0;
          }
          b[r][c] = v;
        }
      }
      int ovf = 0;
      for (int c = 0; c < 128; ++c) ovf |= o32_fexp_bits(mx[c]) > E[c];
      fresh = ovf || len == J->span_max || ch == J->c0;
    }
    if ((fresh || end) && span >= 0) {
      /* drain the span just closed */
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
          const int64_t e = i * 128 + j;
          dd t0 = o32_group_total(g, (int32_t)(uint32_t)acc[e], (int32_t)(uint32_t)acc[16384 + e],
                                  (int32_t)(uint32_t)acc[2 * 16384 + e], (int32_t)(uint32_t)acc[3 * 16384 + e]);
          if (g == 1 && i == j) t0 = dd_add(t0, (dd){(double)s8[i] * 0x1p-16, 0.0}); /* D8 diagonal */
          const int sc = E[i] + E[j] - 92 + base;
          dd t = {scalbn(t0.hi, sc), scalbn(t0.lo, sc)};
          dd* o = &J->P[j * 128 + i];
          if (J->accumulate || span > 0) t = dd_add(*o, t);
          *o = t;
        }
    }
    if (end) break;
    if (fresh) {
      ++span;
      len = 0;
      for (int c = 0; c < 128; ++c) {
        E[c] = mx[c] ? o32_fexp_bits(mx[c]) + O32_HEAD : O32_ZERO_E;
        s8[c] = 0;
      }
      memset(acc, 0, sizeof(int64_t) * 4 * 128 * 128);
    }
    ++len;
    for (int r = 0; r < 64; ++r)
      for (int c = 0; c < 128; ++c) {
        const uint64_t y = o32_fixed48(b[r][c], E[c]);
        for (int p = 1; p <= 6; ++p) D[((p - 1) * 64 + r) * 128 + c] = (int8_t)(((y >> (8 * (6 - p))) & 0xFFu) ^ 0x80u);
        const int d4 = D[(3 * 64 + r) * 128 + c];
        s8[c] += d4 * d4;
      }
    for (int k = 0; k < 6; ++k) {
      int p, q, ai;
      o32_product(g, k, &p, &q, &ai);
      int64_t* A = acc + (int64_t)ai * 16384;
      for (int r = 0; r < 64; ++r) {
        const int8_t* dp = D + ((p - 1) * 64 + r) * 128;
        const int8_t* dq = D + ((q - 1) * 64 + r) * 128;
        for (int i = 0; i < n; ++i) {
          const int64_t x = dp[i];
          if (!x) continue;
          int64_t* row = A + i * 128;
          for (int j = 0; j < n; ++j) row[j] += x * dq[j];
        }
      }
    }
  }
  if (span < 0 && !J->accumulate)
    for (int64_t e = 0; e < 128 * 128; ++e) J->P[e] = (dd){0.0, 0.0};
  free(acc);
  free(D);
  free(b);
  return NULL;
}

int port_gram_f32_ozaki(const float* a, int64_t m, int64_t n, int npairs, int nranges, const int64_t* bounds,
                        int span_max, int threads, double* out) {
  if (m < 1 || n < 1 || n > 128 || npairs < 1 || nranges < 1 || span_max < 1) return ST_INVALID;
  const int ncta = 2 * npairs;
  dd* P = (dd*)calloc((size_t)ncta * 128 * 128, sizeof(dd));
  int* bad = (int*)calloc((size_t)ncta * 128, sizeof(int));
  O32Job* jobs = (O32Job*)malloc(sizeof(O32Job) * (size_t)ncta);
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  for (int l = 0; l < nranges; ++l) {
    const int64_t cb = bounds[l], nall = bounds[l + 1] - bounds[l];
    for (int k = 0; k < ncta; ++k) {
      const int pr = k >> 1;
      jobs[k] = (O32Job){a,     m,      n, cb + nall * pr / npairs, cb + nall * (pr + 1) / npairs, k & 1, l > 0,
                         span_max, P + (int64_t)k * 128 * 128, bad + (int64_t)k * 128};
    }
    for (int k0 = 0; k0 < ncta; k0 += threads) {
      pthread_t th[64];
      const int cnt = ncta - k0 < threads ? ncta - k0 : threads;
      for (int t = 0; t < cnt; ++t) pthread_create(&th[t], NULL, o32_worker, &jobs[k0 + t]);
      for (int t = 0; t < cnt; ++t) pthread_join(th[t], NULL);
    }
  }
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i <= j; ++i) {
      dd acc = {0.0, 0.0};
      int isbad = 0;
      for (int k = 0; k < ncta; ++k) {
        acc = dd_add(acc, P[(int64_t)k * 16384 + j * 128 + i]);
        acc = dd_add(acc, P[(int64_t)k * 16384 + i * 128 + j]);
        isbad |= bad[k * 128 + i] | bad[k * 128 + j];
      }
      const double v = isbad ? NAN : acc.hi;
      out[j * n + i] = v;
      out[i * n + j] = v;
    }
  free(P);
  free(bad);
  free(jobs);
  return ST_OK;
}
