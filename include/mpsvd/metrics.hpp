// Measured error quantities of a thin SVD, the subset of
// proj/include/mpsvd/metrics.hpp that validates the hot path at scale:
// the singular-value error and the row-wise backward error. The backward
// error runs on the GPU (csrc/metrics.cu) so a 2^26-row factorisation can be
// checked where it lives; the reference evaluates it on the CPU.
#pragma once

#include <vector>

#include "mpsvd/types.hpp"

namespace mpsvd {

// proj/include/mpsvd/metrics.hpp:44-47
struct BackwardErrorReport {
  double max_rel = 0.0;
  index_t skipped_rows = 0;  // rows of A with exactly zero norm
};

// max_i |computed_i - reference_i| / reference_i (proj/src/metrics.cpp:26-38).
// Throws InvalidArgument on a length mismatch or a non-positive reference
// entry (message names the 1-based index, like the reference).
double max_rel_sv_error(const std::vector<double>& computed, const std::vector<double>& reference);

// max_i ||(U diag(sigma) V^T - A)(i,:)|| / ||A(i,:)|| with U and V widened
// to binary64, W = U diag(sigma) rounded, then W V^T accumulated in binary64
// (proj/src/metrics.cpp:40-70; the summation order inside a row differs,
// within binary64 rounding). Zero rows of A are skipped and counted.
// Throws InvalidArgument when the factor shapes do not match A.
BackwardErrorReport rowwise_backward_error(const DenseMatrix& a, const DenseMatrix& u,
                                           const std::vector<double>& sigma, const DenseMatrix& v);

}  // namespace mpsvd
