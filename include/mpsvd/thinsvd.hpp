// mpsvd-b200 public C++ API for the Gram-based thin SVD — the reference's
// proj/include/mpsvd/jacobi.hpp:29-52 (JacobiConfig, SvdFactors, EigFactors,
// JacobiStats) and proj/include/mpsvd/thinsvd.hpp:20-59 (EigensolverChoice,
// PhaseTimes, ThinSvdResult, mp_thin_svd), executed on an sm_100a GPU.
//
//   mp_thin_svd       drop-in for thinsvd.hpp:58-59 (fp32 A; Gram + Jacobi in
//                     fp64; U in fp32). Rejects fp64 input like the reference
//                     (thinsvd.cpp:52-53).
//   mp_thin_svd_f64   ADDITIVE: fp64 A; Gram + Jacobi in double-double; U fp64.
//   twosided_jacobi_eig  drop-in for jacobi.hpp:45-46 (fp64 M), on the GPU.
//
// Every EigensolverChoice runs on the GPU: TwoSidedJacobi (K4/K5), and the
// GramCholSvd / OneSidedJacobiOnGram branches of thinsvd.cpp:37-47,90-104
// (Cholesky K8 + one-sided Jacobi K9, csrc/onesided.cu), binary32 A only.
#pragma once

#include <vector>

#include "mpsvd/types.hpp"

namespace mpsvd {

struct JacobiConfig {
  double tol = 0.0;     // 0: n * u(precision of M); u_dd = 2^-104 for double-double
  int max_sweeps = 30;  // NoConvergenceError beyond this
};

// Default for the double-double path (ADDITIVE). Two-sided Jacobi needs more
// sweeps to reach tol = n * 2^-104 on ill-conditioned, non-graded Grams (the
// BASELINE C5 matrices: ~30 sweeps at n = 128, ~37 at n = 256), so the
// cap is 100 instead of the fp64 path's 30.
constexpr int kDdMaxSweeps = 100;
inline JacobiConfig dd_jacobi_config() {
  JacobiConfig c;
  c.max_sweeps = kDdMaxSweeps;
  return c;
}

struct SvdFactors {
  DenseMatrix u;
  std::vector<double> sigma;  // descending, exact in `precision`
  DenseMatrix v;
  Precision precision = Precision::Working;
};

struct EigFactors {
  DenseMatrix v;
  std::vector<double> lambda;  // descending
  Precision precision = Precision::Higher;
};

struct JacobiStats {
  int sweeps = 0;
  long rotations = 0;
  long pairs_per_sweep = 0;
};

enum class EigensolverChoice { TwoSidedJacobi, GramCholSvd, OneSidedJacobiOnGram };

// Seconds. gram/eigen/compute_u are device time (CUDA events); overlap is the
// remainder of the wall-clock total (host<->device copies, setup), so the
// four partition `total` exactly as in the reference (thinsvd.hpp:28-38).
struct PhaseTimes {
  double gram = 0.0;
  double eigen = 0.0;
  double compute_u = 0.0;
  double overlap = 0.0;
  double total = 0.0;
};

struct ThinSvdResult {
  SvdFactors factors;
  EigensolverChoice eigensolver = EigensolverChoice::TwoSidedJacobi;
  bool qr_baseline = false;
  PhaseTimes times;
  int gram_sync_events = 0;  // 1: one global combine of the partial Grams
  index_t gram_blocks = 0;   // logical row blocks combined by the fixed tree
  // device instrumentation (additive)
  int jacobi_sweeps = 0;
  long jacobi_rotations = 0;
};

ThinSvdResult mp_thin_svd(const DenseMatrix& a, EigensolverChoice choice,
                          const JacobiConfig& cfg = {}, int threads = 1);

ThinSvdResult mp_thin_svd_f64(const DenseMatrix& a, const JacobiConfig& cfg = dd_jacobi_config(),
                              int threads = 1);

// proj/include/mpsvd/thinsvd.hpp:67-75: Gram (K1) and Cholesky (K8) in
// binary64, R cast to binary32 (with the cast's overflow checks), then every
// row of Q from Q(i,:) R = A(i,:) by forward substitution in binary32 (K10,
// the reference's operation order). NotPositiveDefiniteError(pivot, value).
struct CholQrFactors {
  DenseMatrix q;
  DenseMatrix r;
};
CholQrFactors mp_cholesky_qr(const DenseMatrix& a);

EigFactors twosided_jacobi_eig(const DenseMatrix& m, const JacobiConfig& cfg = {},
                               JacobiStats* stats = nullptr);

// ||Q^T Q - I||_F accumulated in binary64 (proj/include/mpsvd/dense.hpp:39-40),
// with Q^T Q formed by the fp64 SYRK kernel.
double orth_error(const DenseMatrix& q);

}  // namespace mpsvd
