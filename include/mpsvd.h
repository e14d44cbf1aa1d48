/* mpsvd-b200 — C ABI of the B200 (sm_100a) Gram-based thin SVD.
 *
 * Drop-in for the thin-SVD surface of the reference's C header
 * (proj/include/mpsvd.h): same type names, enum values, function names,
 * argument meaning, ownership rules (caller-owned handles released with
 * *_destroy; accessors borrow) and thread-local diagnostics. Each declaration
 * below cites the reference line it replaces. Declarations marked ADDITIVE do
 * not exist in the reference: the double-double fp64 path, the device-pointer
 * plan API used for benchmarking and multi-GPU, and stage-level entry points
 * used by the parity tests. No declaration exposes a C++ or torch type.
 */
#ifndef MPSVD_B200_H
#define MPSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/include/mpsvd.h:25-37 */
typedef enum mpsvd_status {
  MPSVD_OK = 0,
  MPSVD_ERR_INVALID_ARGUMENT = 1,
  MPSVD_ERR_NOT_POSITIVE_DEFINITE = 2,
  MPSVD_ERR_NO_CONVERGENCE = 3,
  MPSVD_ERR_ZERO_COLUMN = 4,
  MPSVD_ERR_ZERO_DIVISOR = 5,
  MPSVD_ERR_CAST_OVERFLOW = 6,
  MPSVD_ERR_TINY_SINGULAR_VALUE = 7,
  MPSVD_ERR_INFEASIBLE = 8,
  MPSVD_ERR_IO = 9,
  MPSVD_ERR_INTERNAL = 10
} mpsvd_status;

/* proj/include/mpsvd.h:39-42 */
typedef enum mpsvd_precision { MPSVD_PRECISION_WORKING = 0, MPSVD_PRECISION_HIGHER = 1 } mpsvd_precision;

/* proj/include/mpsvd.h:44-48 (every branch runs on the GPU path) */
typedef enum mpsvd_eigensolver {
  MPSVD_EIG_TWOSIDED_JACOBI = 0,
  MPSVD_EIG_GRAM_CHOL_SVD = 1,
  MPSVD_EIG_ONESIDED_JACOBI_GRAM = 2
} mpsvd_eigensolver;

typedef struct mpsvd_matrix mpsvd_matrix;         /* proj/include/mpsvd.h:50 */
typedef struct mpsvd_svd_result mpsvd_svd_result; /* proj/include/mpsvd.h:52 */

/* ---- diagnostics --------------------------------------------------------- */
const char* mpsvd_last_error_message(void); /* proj/include/mpsvd.h:57 */
int64_t mpsvd_last_error_index(void);       /* proj/include/mpsvd.h:60 */

/* ---- matrices (host, column-major) --------------------------------------- */
mpsvd_status mpsvd_matrix_create(int64_t rows, int64_t cols, mpsvd_precision prec,
                                 mpsvd_matrix** out);                        /* mpsvd.h:64-65 */
void mpsvd_matrix_destroy(mpsvd_matrix* a);                                  /* mpsvd.h:66 */
int64_t mpsvd_matrix_rows(const mpsvd_matrix* a);                            /* mpsvd.h:68 */
int64_t mpsvd_matrix_cols(const mpsvd_matrix* a);                            /* mpsvd.h:69 */
mpsvd_precision mpsvd_matrix_precision(const mpsvd_matrix* a);               /* mpsvd.h:70 */
mpsvd_status mpsvd_matrix_set(mpsvd_matrix* a, int64_t row, int64_t col, double value); /* :72 */
mpsvd_status mpsvd_matrix_get(const mpsvd_matrix* a, int64_t row, int64_t col,
                              double* value);                                /* mpsvd.h:73-74 */
int mpsvd_matrix_bitwise_equal(const mpsvd_matrix* a, const mpsvd_matrix* b); /* mpsvd.h:77 */
/* ADDITIVE: borrowed pointer to the column-major storage (float* or double*),
 * page-locked when possible; lets a binding fill/read a matrix in one copy. */
void* mpsvd_matrix_data(mpsvd_matrix* a);
/* ||A^T A - I||_F in binary64 (mpsvd.h:85), A^T A formed on the GPU. */
mpsvd_status mpsvd_orth_error(const mpsvd_matrix* a, double* out);
/* max_i |computed_i - reference_i| / reference_i (mpsvd.h:147-148,
 * metrics.cpp:26-38); MPSVD_ERR_INVALID_ARGUMENT on a non-positive reference. */
mpsvd_status mpsvd_max_rel_sv_error(const double* computed, const double* reference, int64_t count,
                                    double* out);
/* max_i ||(U diag(sigma) V^T - A)(i,:)|| / ||A(i,:)|| in binary64, zero rows
 * skipped and counted (mpsvd.h:150-153, metrics.cpp:40-70); on the GPU. */
mpsvd_status mpsvd_rowwise_backward_error(const mpsvd_matrix* a, const mpsvd_matrix* u,
                                          const double* sigma, int64_t count, const mpsvd_matrix* v,
                                          double* max_rel, int64_t* skipped_rows);
/* ADDITIVE: the same on device-resident factors (column-major, leading
 * dimensions lda/ldu >= m, ldv >= n; prec selects float/double storage of
 * A, U, V; d_sigma: n doubles). Synchronous on `stream` (NULL: legacy). */
mpsvd_status mpsvd_backward_error_device(mpsvd_precision prec, const void* d_a, int64_t lda, const void* d_u,
                                         int64_t ldu, const double* d_sigma, const void* d_v, int64_t ldv,
                                         int64_t m, int64_t n, void* stream, double* max_rel,
                                         int64_t* skipped_rows);

/* ---- thin SVD -------------------------------------------------------------- */
/* proj/include/mpsvd.h:116-117: f32 A (m >= n >= 1), Gram + Jacobi in fp64,
 * U in f32. `threads` must be >= 1 (it does not change any bit). */
mpsvd_status mpsvd_thin_svd(const mpsvd_matrix* a, mpsvd_eigensolver eig, int threads,
                            mpsvd_svd_result** out);
/* proj/include/mpsvd.h:136-139: mixed-precision Cholesky QR. Gram and
 * Cholesky in binary64, R cast to binary32, row-wise forward substitution in
 * binary32 (thinsvd.cpp:125-154); new Working matrices Q (m x n), R (n x n). */
mpsvd_status mpsvd_cholesky_qr(const mpsvd_matrix* a, mpsvd_matrix** q_out, mpsvd_matrix** r_out);
/* ADDITIVE: f64 A, Gram + Jacobi in double-double, U in f64. */
mpsvd_status mpsvd_thin_svd_f64(const mpsvd_matrix* a, int threads, mpsvd_svd_result** out);

void mpsvd_svd_destroy(mpsvd_svd_result* r);                                 /* mpsvd.h:122 */
const mpsvd_matrix* mpsvd_svd_u(const mpsvd_svd_result* r);                  /* mpsvd.h:124 */
const mpsvd_matrix* mpsvd_svd_v(const mpsvd_svd_result* r);                  /* mpsvd.h:125 */
const double* mpsvd_svd_sigma(const mpsvd_svd_result* r, int64_t* count);    /* mpsvd.h:126 */
void mpsvd_svd_times(const mpsvd_svd_result* r, double times[5]);            /* mpsvd.h:131 */
int mpsvd_svd_sync_events(const mpsvd_svd_result* r);                        /* mpsvd.h:132 */
int64_t mpsvd_svd_gram_blocks(const mpsvd_svd_result* r);                    /* mpsvd.h:133 */
int mpsvd_svd_is_qr_baseline(const mpsvd_svd_result* r);                     /* mpsvd.h:134 */
/* ADDITIVE: Jacobi sweeps / rotations of the solve. */
void mpsvd_svd_jacobi_stats(const mpsvd_svd_result* r, int* sweeps, int64_t* rotations);

/* ---- ADDITIVE: device-resident plans (bench / multi-GPU) ------------------ */
/* One plan per (rows, cols, precision, rank): owns every device workspace so
 * mpsvd_plan_execute allocates nothing. Pointers are device pointers on the
 * plan's device; `stream` is a cudaStream_t (NULL = the plan's own stream).
 * m_local rows of A live on this rank; the Gram partials of all ranks are
 * exchanged once through `comm` (NULL: single GPU): an NCCL all-gather, then
 * every rank adds the ranks' partials along the reference's fixed tree
 * (binary64 adds for fp64, dd_add for double-double), so all ranks hold the
 * same bits; MPSVD_F64_EXCHANGE=allreduce uses an NCCL sum for fp64.
 * The host-buffer entry points (mpsvd_thin_svd, mpsvd_thin_svd_f64) shard
 * over the visible GPUs by themselves (MPSVD_DEVICES). */
typedef struct mpsvd_comm mpsvd_comm;
typedef struct mpsvd_plan mpsvd_plan;

typedef struct mpsvd_exec_info {
  int status;          /* mpsvd_status of the device pipeline */
  int64_t error_index; /* 1-based index of the failure (0: none) */
  double error_value;
  int sweeps;
  int64_t rotations;
  double ms_gram, ms_eigen, ms_compute_u; /* CUDA-event device times */
  int kernel_launches; /* kernels of this library launched by one execute */
  int64_t rounds;      /* parallel Jacobi rounds executed (two-sided solver) */
  int gram_kernel;     /* Gram kernel of the last execute: 0 K1 (DMMA), 1 K1z (int8 Ozaki),
                          2 K2 (Dot2), 3 K2z (int8 Ozaki) */
  int av_kernel;       /* U = A W kernel: 0 av_kernel (SIMT), 1 av_tc_f32 (tcgen05), 2 av_dmma_f64,
                          -1 none */
} mpsvd_exec_info;

mpsvd_status mpsvd_comm_unique_id(unsigned char id[128]);
mpsvd_status mpsvd_comm_init(const unsigned char id[128], int nranks, int rank, mpsvd_comm** out);
void mpsvd_comm_destroy(mpsvd_comm* c);

mpsvd_status mpsvd_plan_create(int64_t m_local, int64_t n, mpsvd_precision working, mpsvd_comm* comm,
                               mpsvd_plan** out);
/* d_a: m_local x n column-major (lda >= m_local); d_u: m_local x n (ldu);
 * d_sigma: n doubles (device); d_v: n x n working precision (device).
 * Asynchronous; completes on `stream`. */
mpsvd_status mpsvd_plan_execute(mpsvd_plan* p, const void* d_a, int64_t lda, void* d_u, int64_t ldu,
                                void* d_sigma, void* d_v, void* stream);
/* Spectral branch of later executes (default MPSVD_EIG_TWOSIDED_JACOBI; the
 * one-sided branches need a MPSVD_PRECISION_WORKING plan). */
mpsvd_status mpsvd_plan_set_eigensolver(mpsvd_plan* p, mpsvd_eigensolver eig);
/* Cholesky QR of device-resident A (binary32 plan): Q (ldq >= m_local), R
 * (n x n binary32, may be NULL) on `stream`; complete with mpsvd_plan_wait.
 * Multi-rank plans all-reduce the Gram; Q stays row-sharded. */
mpsvd_status mpsvd_plan_cholesky_qr(mpsvd_plan* p, const void* d_a, int64_t lda, void* d_q, int64_t ldq,
                                    float* d_r, void* stream);
/* ADDITIVE: ||Q^T Q - I||_F in binary64 (proj/src/dense.cpp:250-272) of a
 * device-resident m_local x n Q in the plan's precision, Q^T Q formed by the
 * plan's own Gram stage (K1 for binary32, the double-double Gram for
 * binary64) and, on a multi-rank plan, combined over the ranks (a global
 * orthogonality error; every rank must call it). Overwrites the plan's Gram
 * workspace; synchronous on `stream`. */
mpsvd_status mpsvd_plan_orth_error(mpsvd_plan* p, const void* d_q, int64_t ldq, void* stream, double* out);
/* Blocks until the last execute finished; reports the device status. */
mpsvd_status mpsvd_plan_wait(mpsvd_plan* p, mpsvd_exec_info* info);
/* Timed region helpers for the dominant kernels (CUDA events, ms). */
void mpsvd_plan_destroy(mpsvd_plan* p);

/* Text wire format (proj/include/mpsvd.h:79-82): "m n f32|f64" header, then
 * the column-major entries as shortest round-trip decimals, one column per
 * line, so write-then-read is bit-exact. MPSVD_ERR_IO on a bad header, tag,
 * short body, unparsable value or an unopenable file. Host-only. */
mpsvd_status mpsvd_matrix_write_file(const char* path, const mpsvd_matrix* a);
mpsvd_status mpsvd_matrix_read_file(const char* path, mpsvd_matrix** out);

/* ---- ADDITIVE: stage entry points (host buffers; parity tests) ------------- */
/* M = A^T A: prec WORKING -> f32 A, fp64 M (m_hi); HIGHER -> f64 A,
 * double-double M (m_hi + m_lo). */
mpsvd_status mpsvd_stage_gram(mpsvd_precision prec, const void* a, int64_t m, int64_t n, double* m_hi,
                              double* m_lo);
/* The double-double Gram schedule of an m x n plan: *ozaki = 1 when the
 * int8 tensor-core Gram (K2z) runs; split s covers 32-row chunks
 * [scb[s], scb[s + 1]); logical block b holds splits [bsb[b], bsb[b + 1]).
 * cap bounds both arrays. */
mpsvd_status mpsvd_stage_gram_schedule(int64_t m, int64_t n, int cap, int* nsplit, int* nblocks, int* scb,
                                       int* bsb, int* ozaki);
/* The binary32 Gram schedule of an m x n plan: *ozaki = 1 when K1z (the int8
 * tensor-core Gram, gram_ozaki32.cu) runs; it then launches once per range
 * [bounds[b], bounds[b + 1]) of 32-row chunks (b < *nbounds - 1) with
 * *npairs CTA pairs. cap bounds `bounds`. */
mpsvd_status mpsvd_stage_gram32_schedule(int64_t m, int64_t n, int cap, int* ozaki, int* npairs, int* nbounds,
                                         int64_t* bounds);
/* Two-sided Jacobi on the GPU: dd = 0 fp64 (m_lo ignored), 1 double-double.
 * Outputs sorted/sign-fixed eigenpairs in the higher precision. */
mpsvd_status mpsvd_stage_jacobi(int dd, const double* m_hi, const double* m_lo, int64_t n, double tol,
                                int max_sweeps, double* lam_hi, double* lam_lo, double* v_hi,
                                double* v_lo, int* sweeps, int64_t* rotations);

/* Spectral phase of MPSVD_EIG_GRAM_CHOL_SVD / MPSVD_EIG_ONESIDED_JACOBI_GRAM on
 * a binary64 Gram m_hi (n x n): Cholesky + binary32 one-sided Jacobi of R, or
 * binary64 one-sided Jacobi of M (thinsvd.cpp:37-47,90-104); outputs the
 * sorted working-precision sigma and sign-fixed binary32 V. */
mpsvd_status mpsvd_stage_onesided(mpsvd_eigensolver eig, const double* m_hi, int64_t n, double tol,
                                  int max_sweeps, double* sigma, float* v, int* sweeps, int64_t* rotations);

/* The multi-GPU exchange's combine (the kernel Plan::exchange runs after the
 * all-gather) on nranks partial Grams supplied from the host, on one GPU:
 * part_hi (and, for HIGHER, part_lo) hold nranks consecutive n x n
 * column-major matrices; M = the reference tree over ranks ((0,1),(2,3),...
 * then doubling widths, parallel_gram.cpp:93-102) with binary64 adds
 * (WORKING plans' fp64 Gram) or dd_add (HIGHER). 1 <= nranks <= 16. */
mpsvd_status mpsvd_stage_rank_combine(mpsvd_precision prec, const double* part_hi, const double* part_lo, int nranks,
                                      int64_t n, double* m_hi, double* m_lo);

/* ---- formatting (proj/include/mpsvd.h:166-171) ----------------------------- */
/* Shortest decimal string that parses back to the identical double; returns
 * the full length (excluding NUL), truncating to cap - 1 characters; a cap of
 * 32 always suffices. Host-only. */
size_t mpsvd_format_shortest(double value, char* buf, size_t cap);

/* ---- ADDITIVE: measured device peaks (roofline denominators) --------------- */
double mpsvd_fp64_peak_tflops(int device);
/* 1 if a CUDA device is usable by this library. */
int mpsvd_device_available(void);

#ifdef __cplusplus
}
#endif
#endif /* MPSVD_B200_H */
