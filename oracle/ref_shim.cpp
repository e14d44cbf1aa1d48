// TEST INFRASTRUCTURE ONLY. Flat extern "C" surface over the UNMODIFIED
// reference library (compiled in place from /root/reference/proj by
// oracle/Makefile into oracle/_ref/libmpsvd_ref.so). Only tests/, smoke() and
// bench.py's reference / cpu_baseline legs load it, and only as the checker.
//
// Every function takes raw column-major buffers (index j*rows+i, like
// proj/include/mpsvd/types.hpp:175-177) and returns an mpsvd_status code
// (proj/include/mpsvd.h:25-37); the 1-based error index / value of the last
// failure is kept thread-locally and read back with refx_last_error().
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "mpsvd/dense.hpp"
#include "mpsvd/jacobi.hpp"
#include "mpsvd/matgen.hpp"
#include "mpsvd/metrics.hpp"
#include "mpsvd/parallel_gram.hpp"
#include "mpsvd/thinsvd.hpp"
#include "mpsvd/types.hpp"
#include "support/dd.hpp"

using namespace mpsvd;

namespace {

thread_local std::string t_msg;
thread_local int64_t t_index = 0;
thread_local double t_value = 0.0;

template <typename F>
int run(F&& body) noexcept {
  t_msg.clear();
  t_index = 0;
  t_value = 0.0;
  try {
    body();
    return 0;
  } catch (const InvalidArgument& e) {
    t_msg = e.what();
    return 1;
  } catch (const NotPositiveDefiniteError& e) {
    t_msg = e.what();
    t_index = e.pivot;
    t_value = e.value;
    return 2;
  } catch (const NoConvergenceError& e) {
    t_msg = e.what();
    t_index = e.sweeps;
    t_value = e.max_offdiag;
    return 3;
  } catch (const ZeroColumnError& e) {
    t_msg = e.what();
    t_index = e.column;
    return 4;
  } catch (const ZeroDivisorError& e) {
    t_msg = e.what();
    t_index = e.index;
    return 5;
  } catch (const CastOverflowError& e) {
    t_msg = e.what();
    return 6;
  } catch (const TinySingularValueError& e) {
    t_msg = e.what();
    t_index = e.index;
    t_value = e.value;
    return 7;
  } catch (const IoError& e) {
    t_msg = e.what();
    return 9;
  } catch (const std::exception& e) {
    t_msg = e.what();
    return 10;
  }
}

DenseMatrix from_f32(const float* a, int64_t m, int64_t n) {
  DenseMatrix out(m, n, Precision::Working);
  std::memcpy(out.fptr(), a, sizeof(float) * static_cast<size_t>(m * n));
  return out;
}

DenseMatrix from_f64(const double* a, int64_t m, int64_t n) {
  DenseMatrix out(m, n, Precision::Higher);
  std::memcpy(out.dptr(), a, sizeof(double) * static_cast<size_t>(m * n));
  return out;
}

}  // namespace

extern "C" {

const char* refx_last_error(int64_t* index, double* value) {
  if (index) *index = t_index;
  if (value) *value = t_value;
  return t_msg.c_str();
}

// mp_thin_svd (proj/src/thinsvd.cpp:49-123) on an f32 column-major m x n A.
int refx_thin_svd(const float* a, int64_t m, int64_t n, int choice, int threads,
                  float* u, double* sigma, float* v, double* times5,
                  int* sync_events, int64_t* gram_blocks) {
  return run([&] {
    const auto A = from_f32(a, m, n);
    const auto r = mp_thin_svd(A, static_cast<EigensolverChoice>(choice), {}, threads);
    std::memcpy(u, r.factors.u.fptr(), sizeof(float) * static_cast<size_t>(m * n));
    std::memcpy(v, r.factors.v.fptr(), sizeof(float) * static_cast<size_t>(n * n));
    std::memcpy(sigma, r.factors.sigma.data(), sizeof(double) * static_cast<size_t>(n));
    if (times5) {
      times5[0] = r.times.gram;
      times5[1] = r.times.eigen;
      times5[2] = r.times.compute_u;
      times5[3] = r.times.overlap;
      times5[4] = r.times.total;
    }
    if (sync_events) *sync_events = r.gram_sync_events;
    if (gram_blocks) *gram_blocks = r.gram_blocks;
  });
}

// Precision-checked entry: a Higher (f64) matrix must be rejected
// (proj/src/thinsvd.cpp:52-53).
int refx_thin_svd_f64_input(const double* a, int64_t m, int64_t n) {
  return run([&] {
    const auto A = from_f64(a, m, n);
    (void)mp_thin_svd(A, EigensolverChoice::TwoSidedJacobi);
  });
}

// partitioned_gram (proj/src/parallel_gram.cpp:79-112) of cast(A, Higher).
int refx_partitioned_gram_f32(const float* a, int64_t m, int64_t n, int workers,
                              int64_t blocks, double* out, int* sync_events,
                              int64_t* nblocks) {
  return run([&] {
    const auto ah = cast(from_f32(a, m, n), Precision::Higher);
    GramRunStats st;
    const auto g = partitioned_gram(ah, workers, blocks, &st);
    std::memcpy(out, g.dptr(), sizeof(double) * static_cast<size_t>(n * n));
    if (sync_events) *sync_events = st.sync_events;
    if (nblocks) *nblocks = st.blocks;
  });
}

int refx_partitioned_gram_f64(const double* a, int64_t m, int64_t n, int workers,
                              int64_t blocks, double* out) {
  return run([&] {
    const auto g = partitioned_gram(from_f64(a, m, n), workers, blocks, nullptr);
    std::memcpy(out, g.dptr(), sizeof(double) * static_cast<size_t>(n * n));
  });
}

// dense gram (proj/src/dense.cpp:179-187) in A's own precision, f64 here.
int refx_gram_f64(const double* a, int64_t m, int64_t n, double* out) {
  return run([&] {
    const auto g = gram(from_f64(a, m, n));
    std::memcpy(out, g.dptr(), sizeof(double) * static_cast<size_t>(n * n));
  });
}

// twosided_jacobi_eig (proj/src/jacobi.cpp:268-311) on an f64 symmetric M.
int refx_twosided_jacobi(const double* mtx, int64_t n, double tol, int max_sweeps,
                         double* lambda, double* v, int* sweeps, int64_t* rotations) {
  return run([&] {
    JacobiConfig cfg;
    cfg.tol = tol;
    cfg.max_sweeps = max_sweeps;
    JacobiStats st;
    const auto e = twosided_jacobi_eig(from_f64(mtx, n, n), cfg, &st);
    std::memcpy(lambda, e.lambda.data(), sizeof(double) * static_cast<size_t>(n));
    std::memcpy(v, e.v.dptr(), sizeof(double) * static_cast<size_t>(n * n));
    if (sweeps) *sweeps = st.sweeps;
    if (rotations) *rotations = st.rotations;
  });
}

// reference_svd (proj/src/metrics.cpp:103-105): f64 one-sided Jacobi of A.
int refx_reference_svd_f32(const float* a, int64_t m, int64_t n, double* sigma) {
  return run([&] {
    const auto s = reference_svd(from_f32(a, m, n));
    std::memcpy(sigma, s.data(), sizeof(double) * static_cast<size_t>(n));
  });
}

int refx_reference_svd_f64(const double* a, int64_t m, int64_t n, double* sigma) {
  return run([&] {
    const auto s = reference_svd(from_f64(a, m, n));
    std::memcpy(sigma, s.data(), sizeof(double) * static_cast<size_t>(n));
  });
}

// orth_error (proj/src/dense.cpp:250-272).
int refx_orth_error_f32(const float* q, int64_t m, int64_t n, double* out) {
  return run([&] { *out = orth_error(from_f32(q, m, n)); });
}

int refx_orth_error_f64(const double* q, int64_t m, int64_t n, double* out) {
  return run([&] { *out = orth_error(from_f64(q, m, n)); });
}

// mp_cholesky_qr (proj/src/thinsvd.cpp:125-154).
int refx_cholesky_qr(const float* a, int64_t m, int64_t n, float* q, float* r) {
  return run([&] {
    const auto f = mp_cholesky_qr(from_f32(a, m, n));
    std::memcpy(q, f.q.fptr(), sizeof(float) * static_cast<size_t>(m * n));
    std::memcpy(r, f.r.fptr(), sizeof(float) * static_cast<size_t>(n * n));
  });
}

// rowwise_backward_error / max_rel_sv_error (proj/src/metrics.cpp:26-70):
// A, U, V in Working (f32) storage, the thin-SVD factors' layout.
int refx_rowwise_backward_error_f32(const float* a, const float* u, const double* sigma, const float* v,
                                    int64_t m, int64_t n, double* max_rel, int64_t* skipped) {
  return run([&] {
    const auto rep = rowwise_backward_error(from_f32(a, m, n), from_f32(u, m, n),
                                            std::vector<double>(sigma, sigma + n), from_f32(v, n, n));
    *max_rel = rep.max_rel;
    *skipped = rep.skipped_rows;
  });
}

int refx_rowwise_backward_error_f64(const double* a, const double* u, const double* sigma, const double* v,
                                    int64_t m, int64_t n, double* max_rel, int64_t* skipped) {
  return run([&] {
    const auto rep = rowwise_backward_error(from_f64(a, m, n), from_f64(u, m, n),
                                            std::vector<double>(sigma, sigma + n), from_f64(v, n, n));
    *max_rel = rep.max_rel;
    *skipped = rep.skipped_rows;
  });
}

int refx_max_rel_sv_error(const double* computed, const double* reference, int64_t count, double* out) {
  return run([&] {
    *out = max_rel_sv_error(std::vector<double>(computed, computed + count),
                            std::vector<double>(reference, reference + count));
  });
}

// build_problem (proj/src/matgen.cpp:266-289): the acceptance-grid generator.
int refx_build_problem(int64_t m, int64_t n, double kappa_d, double kappa_b,
                       int matrix_id, uint64_t seed, float* a, double* sigma_ref,
                       double* realized_kappa_b) {
  return run([&] {
    TestMatrixSpec s{m, n, kappa_d, kappa_b, matrix_id, seed};
    const auto p = build_problem(s);
    std::memcpy(a, p.a.fptr(), sizeof(float) * static_cast<size_t>(m * n));
    std::memcpy(sigma_ref, p.sigma_ref.data(), sizeof(double) * static_cast<size_t>(n));
    *realized_kappa_b = p.realized_kappa_b;
  });
}

// haar_orthonormal (proj/src/matgen.cpp:94-108) with Rng(seed).
int refx_haar_orthonormal(int64_t m, int64_t n, uint64_t seed, double* q) {
  return run([&] {
    Rng rng(seed);
    const auto h = haar_orthonormal(m, n, rng);
    std::memcpy(q, h.dptr(), sizeof(double) * static_cast<size_t>(m * n));
  });
}

// ddtest::dd_gram (proj/tests/support/dd.cpp:75-88) of an f64 matrix.
int refx_dd_gram(const double* a, int64_t m, int64_t n, double* hi, double* lo) {
  return run([&] {
    const auto g = ddtest::dd_gram(from_f64(a, m, n));
    for (size_t k = 0; k < g.size(); ++k) {
      hi[k] = g[k].hi;
      lo[k] = g[k].lo;
    }
  });
}

// ddtest::oracle_eigenvalues / oracle_singular_values (dd.cpp:155-176):
// LDL^T inertia bisection in double-double, n <= 16.
int refx_dd_oracle_eigenvalues(const double* mtx, int64_t n, double* out) {
  return run([&] {
    const auto l = ddtest::oracle_eigenvalues(from_f64(mtx, n, n));
    std::memcpy(out, l.data(), sizeof(double) * static_cast<size_t>(n));
  });
}

int refx_dd_oracle_singular_values_f64(const double* a, int64_t m, int64_t n, double* out) {
  return run([&] {
    const auto s = ddtest::oracle_singular_values(from_f64(a, m, n));
    std::memcpy(out, s.data(), sizeof(double) * static_cast<size_t>(n));
  });
}

int refx_dd_oracle_singular_values_f32(const float* a, int64_t m, int64_t n, double* out) {
  return run([&] {
    const auto s = ddtest::oracle_singular_values(from_f32(a, m, n));
    std::memcpy(out, s.data(), sizeof(double) * static_cast<size_t>(n));
  });
}

}  // extern "C"
