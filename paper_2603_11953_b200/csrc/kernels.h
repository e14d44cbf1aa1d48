// Launchers of the sm_100a kernels (host-callable; implemented in *.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include <vector>

namespace mpsvd {
namespace dev {

struct DevStatus;

// gram.cu --------------------------------------------------------------------
size_t gram_smem_bytes(bool dd);
// K1: tp_diag / tp_off list the diagonal and off-diagonal tile pairs.
cudaError_t launch_gram_f32(const float* a, long long lda, int n, const int2* tiles, int ntp, const int* tp_diag,
                            int ndiag, const int* tp_off, int noff, const longlong2* splits, int nsplit,
                            double* partials, cudaStream_t st);
cudaError_t launch_gram_dd(const double* a, long long lda, int n, const int2* tiles, int ntp,
                           const longlong2* splits, int nsplit, double2* partials,
                           cudaStream_t st);
// sums: nblocks * ntp * 64 * 64 elements of workspace
cudaError_t launch_gram_combine_f64(const double* partials, int ntp, int n, const int* block_split_begin,
                                    int nblocks, double* sums, double* m_out, cudaStream_t st);
cudaError_t launch_gram_combine_dd(const double2* partials, int ntp, int n, const int* block_split_begin,
                                   int nblocks, double2* sums, double2* m_out, cudaStream_t st);
cudaError_t launch_mirror_upper(double* m, int n, cudaStream_t st);
cudaError_t launch_block_tree(const void* blocks, int nblocks, int n, void* m_out, bool dd,
                              cudaStream_t st);

// gram_ozaki.cu: K2z, the double-double Gram on the int8 tensor cores.
// Splits are whole 32-row chunks: split s holds chunks [scb[s], scb[s + 1]).
// Partial slots: split * ozaki_groups() + group, K2's tile layout.
size_t ozaki_digit_bytes(long long m, int n);
int ozaki_groups();
void ozaki_tiles(int n, std::vector<int2>& tiles);  // (128-column block I, 256-column block J)
cudaError_t launch_gram_ozaki(const double* a, long long lda, long long m, int n, const int* scb_dev,
                              const int* scb_host, int nsplit_total, int s0, int ns, const int2* tiles, int ntiles,
                              int* e_cols, unsigned char* digits, double2* partials, int ntp64, int sm_count,
                              cudaStream_t st);

// gram_ozaki32.cu: K1z, the binary64 Gram of a binary32 A (n <= 128) on the
// int8 tensor cores. A is read by TMA (16-byte aligned, lda % 4 == 0).
// begin() clears the non-finite column flags; every range launch covers
// 32-row chunks [c_begin, c_end) with npairs CTA pairs and adds into the
// 2 npairs double-double partial tiles (accumulate = false: overwrite);
// combine() writes M (both triangles).
bool gram_ozaki32_supported(const float* a, long long lda, long long m, int n);
size_t gram_ozaki32_partial_bytes(int npairs);
int gram_ozaki32_max_pairs();
cudaError_t launch_gram_ozaki32_begin(int* bad_cols, cudaStream_t st);
cudaError_t launch_gram_ozaki32_range(const float* a, long long lda, long long m, int n, long long c_begin,
                                      long long c_end, int npairs, double2* partials, int* bad_cols, bool accumulate,
                                      cudaStream_t st);
cudaError_t launch_gram_ozaki32_combine(const double2* partials, int npairs, int n, const int* bad_cols,
                                        double* m_out, cudaStream_t st);

// jacobi.cu ------------------------------------------------------------------
// A (n x n, full symmetric, column-major; f64 or dd=double2) is overwritten:
// on success its diagonal holds the eigenvalues. The rotation log receives
// (c, s) per pair per round; V is rebuilt from it by launch_jacobi_replay.
struct JacobiWorkspace {
  void* a;            // n*n elements of T
  void* diagbuf;      // 2 * np * 3 elements of T
  void* log;          // max_sweeps * (N-1) * np * 2 elements of T
  void* v;            // n*n elements of T (replay output)
  DevStatus* status;
};
size_t jacobi_log_elems(int n, int max_sweeps);
// *fused_replay is set when the launch also rebuilt V (single-CTA solver with
// co-resident replay CTAs); launch_jacobi_replay is then unnecessary.
cudaError_t launch_jacobi(bool dd, int n, double tol, int max_sweeps, const JacobiWorkspace& ws,
                          int sm_count, cudaStream_t st, bool* fused_replay = nullptr);
cudaError_t launch_jacobi_replay(bool dd, int n, const JacobiWorkspace& ws, cudaStream_t st);

// finish: sort, sign, sigma, V in working precision, W = V / sigma.
// working: 0 = fp32 (sigma = fl32(sqrt(lambda))), 1 = fp64 (sigma = fl64(sqrt_dd(lambda))).
cudaError_t launch_finish(bool dd, int n, const JacobiWorkspace& ws, int* perm, double* lambda_hi,
                          double* lambda_lo, double* sigma, void* v_work, void* w_work,
                          int working_f64, cudaStream_t st, void* v_full = nullptr);

// compute_u.cu ----------------------------------------------------------------

cudaError_t launch_av_f32(const float* a, long long lda, long long m, int n, const float* w,
                          float* u, long long ldu, const DevStatus* status, cudaStream_t st);
// K7 on tcgen05 (compute_u_tc.cu): fp32, n <= 128, m % 4 == 0, lda % 4 == 0,
// 16-byte aligned A. `wplanes` is av_tc_wplanes_bytes(n) of device scratch;
// launch_av_tc_save_diag must have stored the Gram's diagonal in it (A's
// column scales) before the Jacobi overwrites M.
bool av_tc_supported(const float* a, long long lda, long long m, int n, long long ldu);
size_t av_tc_wplanes_bytes(int n);
cudaError_t launch_av_tc_save_diag(const double* gram, int n, void* wplanes, cudaStream_t st);
cudaError_t launch_av_tc_f32(const float* a, long long lda, long long m, int n, const float* w, void* wplanes,
                             float* u, long long ldu, const DevStatus* status, int sm_count, cudaStream_t st,
                             bool prep = true);  // prep: split W into its bf16 pieces first
// K7 fp64 on the DMMA pipe (compute_u.cu)
cudaError_t launch_av_dmma_f64(const double* a, long long lda, long long m, int n, const double* w, double* u,
                               long long ldu, const DevStatus* status, cudaStream_t st);
cudaError_t launch_av_f64(const double* a, long long lda, long long m, int n, const double* w,
                          double* u, long long ldu, const DevStatus* status, cudaStream_t st);

// onesided.cu -----------------------------------------------------------------
// K8: R = chol(M) (fp64, upper; r64 n*n doubles, also the workspace when M
// does not fit in shared memory) and its binary32 image r32 (n*n floats).
cudaError_t launch_chol_upper(const double* m, int n, double* r64, float* r32, DevStatus* status, cudaStream_t st);
// K9: one-sided Jacobi on x (m x n, T = float when f32 else double, rotated
// in place), v: n*n T scratch; sig_raw: n doubles; v_out: n*n doubles;
// aux: onesided_aux_words(max_sweeps) words.
size_t onesided_aux_words(int max_sweeps);
cudaError_t launch_onesided(bool f32, void* x, void* v, int m, int n, double tol, int max_sweeps, DevStatus* status,
                            double* sig_raw, double* v_out, unsigned long long* aux, int sm_count, cudaStream_t st);
// mode 0: GramCholSvd (sigma = sig_raw), 1: OneSidedJacobiOnGram (fl32(sqrt))
cudaError_t launch_onesided_sort(const double* sig_raw, int n, int mode, DevStatus* status, int* perm, double* sigma,
                                 cudaStream_t st);
// finish_columns on an fp64 V (sorted by perm, signed, cast; W = V / sigma)
cudaError_t launch_finish_columns_f64(int n, const double* v, const DevStatus* status, const int* perm,
                                      const double* sigma, void* v_work, void* w_work, int working_f64,
                                      cudaStream_t st);

// cholqr.cu -------------------------------------------------------------------
// K10: Q(i,:) R = A(i,:) by forward substitution per row in binary32 (R: the
// n x n binary32 upper factor, column-major).
cudaError_t launch_cholqr_rows(const float* a, long long lda, long long m, int n, const float* r, float* q,
                               long long ldq, const DevStatus* status, int sm_count, cudaStream_t st);

// metrics.cu ------------------------------------------------------------------
// Row-wise backward error max_i ||(U diag(sigma) V^T - A)(i,:)|| / ||A(i,:)||
// (proj/src/metrics.cpp:40-70) in binary64; f64 selects double storage of
// A, U, V (else float). `partial` holds backward_partial_elems(m, n) doubles;
// out[0] = bit pattern of the maximum, out[1] = zero rows skipped.
size_t backward_partial_elems(long long m, int n);
cudaError_t launch_backward_error(bool f64, const void* a, long long lda, const void* u, long long ldu,
                                  const double* sigma, const void* v, long long ldv, long long m, int n,
                                  double* partial, unsigned long long* out, cudaStream_t st);

// microbench.cu ---------------------------------------------------------------
double measure_fp64_peak_tflops(int device);

}  // namespace dev
}  // namespace mpsvd
