/* TEST INFRASTRUCTURE ONLY — CPU restatement ("port") of the reference's hot
 * path, used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs as the CHECKER. The product (paper_2603_11953_b200)
 * never links, loads or calls this file.
 *
 * Parity status: PINNED. tests/test_oracle_port.py checks this restatement
 * bit-for-bit against the unmodified reference compiled in place
 * (oracle/_ref/libmpsvd_ref.so, see oracle/Makefile) on the fp32 path, and
 * the double-double primitives against the reference's own dd test oracle
 * (proj/tests/support/dd.cpp) and its golden vectors (tests/golden/).
 *
 * Two semantics are restated (argument `sem`):
 *   PORT_SEM_REFERENCE    the reference's cyclic-by-rows sweep with its exact
 *                         formulas (proj/src/jacobi.cpp:189-264) -> bitwise
 *                         equal to the reference;
 *   PORT_SEM_DEVICE       the parallel round-robin schedule and FMA-based
 *                         formulas the CUDA kernels implement,
 *                         so the GPU path can be checked bit-for-bit too.
 * All matrices are column-major, index j*rows+i
 * (proj/include/mpsvd/types.hpp:175-177). Status codes follow
 * proj/include/mpsvd.h:25-37.
 */
#ifndef MPSVD_PORT_H
#define MPSVD_PORT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* sem: which arithmetic to restate (see header comment). */
enum { PORT_SEM_REFERENCE = 0, PORT_SEM_DEVICE = 1 };

typedef struct port_error {
  int status;      /* mpsvd_status */
  int64_t index;   /* 1-based pivot / sigma index (0: none) */
  double value;    /* offending value / worst normalized off-diagonal */
} port_error;

typedef struct port_jacobi_stats {
  int sweeps;
  int64_t rotations;
  int64_t pairs_per_sweep;
} port_jacobi_stats;

/* ---- schedule helpers ---------------------------------------------------- */
int port_partition_plan(int64_t m, int workers, int64_t blocks, int64_t* ranges,
                        int64_t* nblocks);
void port_rr_pair(int64_t n, int64_t round, int64_t k, int64_t* p, int64_t* q);

/* ---- fp64 Gram (fp32 input widened exactly) ------------------------------ */
int port_partitioned_gram_f32(const float* a, int64_t m, int64_t n, int64_t blocks,
                              double* out);
int port_partitioned_gram_f64(const double* a, int64_t m, int64_t n, int64_t blocks,
                              double* out);

/* ---- fp64 two-sided Jacobi ---------------------------------------------- */
int port_twosided_jacobi_f64(const double* mtx, int64_t n, double tol, int max_sweeps,
                             int sem, double* lambda, double* v,
                             port_jacobi_stats* stats, port_error* err);

/* ---- fp32 thin SVD (Algorithm 1) ---------------------------------------- */
int port_thin_svd_f32(const float* a, int64_t m, int64_t n, int threads, int sem,
                      float* u, double* sigma, float* v, double* times5,
                      port_error* err);

int port_av_f32(const float* a, int64_t m, int64_t n, const float* w, float* u, int threads);

/* ---- the one-sided branches (thinsvd.cpp:37-47,90-104) ------------------- */
/* choice: 0 TwoSidedJacobi, 1 GramCholSvd, 2 OneSidedJacobiOnGram */
int port_thin_svd_f32_choice(const float* a, int64_t m, int64_t n, int threads, int sem, int choice,
                             float* u, double* sigma, float* v, double* times5, port_error* err);
/* mixed-precision Cholesky QR (thinsvd.cpp:125-154), reference semantics;
 * the row solve alone (shared by the device K10) */
int port_cholesky_qr_f32(const float* a, int64_t m, int64_t n, float* q, float* r, port_error* err);
void port_cholqr_solve(const float* a, int64_t m, int64_t n, const float* r, float* q);
/* cholesky (dense.cpp:39-58): upper R, strict lower part zero */
int port_cholesky_f64(const double* m, int64_t n, double* r, port_error* err);
/* spectral phase of choice 1 / 2 on the Gram mh: sorted working sigma, V */
int port_onesided_spectral(int choice, const double* mh, int64_t n, double tol, int max_sweeps, int sem,
                           double* sigma, float* v, port_jacobi_stats* stats, port_error* err);

/* ---- double-double ------------------------------------------------------- */
void port_dd_add(double ah, double al, double bh, double bl, double* rh, double* rl);
void port_dd_mul(double ah, double al, double bh, double bl, double* rh, double* rl);
void port_dd_div(double ah, double al, double bh, double bl, double* rh, double* rl);
void port_dd_sqrt(double ah, double al, double* rh, double* rl);

/* G = A^T A, exact products + double-double accumulation (dd.cpp:75-88 order). */
int port_dd_gram(const double* a, int64_t m, int64_t n, int threads, double* hi,
                 double* lo);
/* K2z sub-group i: weight quad (w_hi, nw weights w_hi - k) and steps [pa, pb] */
void port_oz_sub_group(int i, int* whi, int* nw, int* pa, int* pb);
/* K2z (csrc/gram_ozaki.cu) replayed bit for bit on the schedule scb / bsb */
/* K1z (csrc/gram_ozaki32.cu): binary64 Gram of binary32 A (n <= 128) by the
 * int8 Ozaki scheme on the plan's schedule (npairs CTA pairs, chunk ranges
 * bounds[0..nranges]); out: n x n, both triangles. */
int port_gram_f32_ozaki(const float* a, int64_t m, int64_t n, int npairs, int nranges, const int64_t* bounds,
                        int span_max, int threads, double* out);
int port_gram_dd_ozaki(const double* a, int64_t m, int64_t n, int nsplit, const int* scb, int nblocks,
                       const int* bsb, int span_cap, double* out_hi, double* out_lo);
int port_twosided_jacobi_dd(const double* mhi, const double* mlo, int64_t n,
                            double tol, int max_sweeps, int sem, double* lam_hi,
                            double* lam_lo, double* vhi, double* vlo,
                            port_jacobi_stats* stats, port_error* err);
/* fp64-working thin SVD with a double-double Gram + Jacobi (additive API). */
int port_thin_svd_f64dd(const double* a, int64_t m, int64_t n, int threads, int sem,
                        double* u, double* sigma, double* v, double* times5,
                        port_error* err);

/* ---- metrics (evaluated in binary64 / long accumulation) ---------------- */
double port_orth_error_f32(const float* q, int64_t m, int64_t n, int threads);
double port_orth_error_f64(const double* q, int64_t m, int64_t n, int threads);

#ifdef __cplusplus
}
#endif
#endif
