/* A C consumer of the B200 library compiled against the REFERENCE's own C
 * header (proj/include/mpsvd.h, -I /root/reference/proj/include) and linked
 * to libmpsvd_b200.so: proves that a program written for the reference's
 * thin-SVD C surface builds and runs unchanged against this library (same
 * names, enum values, signatures, ownership and error payloads). The same
 * source is also compiled against this repo's include/mpsvd.h (capi_own).
 *
 * The checks restate the reference's C-surface test cases for this path
 * (proj/tests/test_capi.cpp:24-126) as plain C asserts:
 *   matrix lifecycle / precision / bounds        test_capi.cpp:24-41
 *   text round trip, missing file -> IO          test_capi.cpp:43-61
 *   stacked diagonal: sigma = (5, 3) exactly, V = I, U = stacked I,
 *     sync_events == 1, gram_blocks, times partition   test_capi.cpp:63-86
 *   bad eigensolver / threads = 0 -> INVALID_ARGUMENT  test_capi.cpp:99-103
 *   CholQR NPD pivot 2, TinySV index 2 (last_error_*)  test_capi.cpp:106-126
 *   format_shortest (proj/include/mpsvd.h:166-171)
 * Run with --host-only on a machine without a GPU: the host-side calls must
 * work and every compute call must fail with MPSVD_ERR_INTERNAL.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mpsvd.h"

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    ++g_checks;                                                       \
    if (!(cond)) {                                                    \
      ++g_fail;                                                       \
      fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                 \
  } while (0)

static mpsvd_matrix* stacked_diag(int64_t m, const double* d, int64_t n) {
  mpsvd_matrix* a = NULL;
  CHECK(mpsvd_matrix_create(m, n, MPSVD_PRECISION_WORKING, &a) == MPSVD_OK);
  for (int64_t j = 0; j < n; ++j) CHECK(mpsvd_matrix_set(a, j, j, d[j]) == MPSVD_OK);
  return a;
}

static double get(const mpsvd_matrix* a, int64_t i, int64_t j) {
  double v = NAN;
  CHECK(mpsvd_matrix_get(a, i, j, &v) == MPSVD_OK);
  return v;
}

static void host_side(void) {
  mpsvd_matrix* a = NULL;
  CHECK(mpsvd_matrix_create(3, 2, MPSVD_PRECISION_WORKING, &a) == MPSVD_OK);
  CHECK(mpsvd_matrix_rows(a) == 3 && mpsvd_matrix_cols(a) == 2);
  CHECK(mpsvd_matrix_precision(a) == MPSVD_PRECISION_WORKING);
  CHECK(mpsvd_matrix_set(a, 0, 0, 0.1) == MPSVD_OK);
  CHECK(get(a, 0, 0) == (double)0.1f); /* f32 storage rounds, reads widen */
  double v = 0.0;
  CHECK(mpsvd_matrix_get(a, 3, 0, &v) == MPSVD_ERR_INVALID_ARGUMENT);
  CHECK(strlen(mpsvd_last_error_message()) > 0);
  CHECK(mpsvd_matrix_set(NULL, 0, 0, 1.0) == MPSVD_ERR_INVALID_ARGUMENT);
  mpsvd_matrix_destroy(a);

  mpsvd_matrix* b = NULL;
  CHECK(mpsvd_matrix_create(4, 3, MPSVD_PRECISION_HIGHER, &b) == MPSVD_OK);
  for (int64_t j = 0; j < 3; ++j)
    for (int64_t i = 0; i < 4; ++i) CHECK(mpsvd_matrix_set(b, i, j, sin(1.0 + i + 10.0 * j)) == MPSVD_OK);
  const char* path = "capi_ref_roundtrip.txt";
  CHECK(mpsvd_matrix_write_file(path, b) == MPSVD_OK);
  mpsvd_matrix* back = NULL;
  CHECK(mpsvd_matrix_read_file(path, &back) == MPSVD_OK);
  CHECK(back != NULL && mpsvd_matrix_bitwise_equal(b, back) == 1);
  mpsvd_matrix_destroy(back);
  remove(path);
  mpsvd_matrix* missing = NULL;
  CHECK(mpsvd_matrix_read_file("no_such_file_here.txt", &missing) == MPSVD_ERR_IO);
  mpsvd_matrix_destroy(b);

  char buf[32];
  CHECK(mpsvd_format_shortest(0.1, buf, sizeof buf) == 3 && strcmp(buf, "0.1") == 0);
  CHECK(mpsvd_format_shortest(1e-39, buf, sizeof buf) == 5 && strcmp(buf, "1e-39") == 0);
  char small[3];
  CHECK(mpsvd_format_shortest(0.125, small, sizeof small) == 5 && strcmp(small, "0.") == 0);
  CHECK(strtod((mpsvd_format_shortest(1.0 / 3.0, buf, sizeof buf), buf), NULL) == 1.0 / 3.0);

  double s_ref[2] = {2.0, 1.0}, s_got[2] = {2.0, 1.5}, worst = 0.0;
  CHECK(mpsvd_max_rel_sv_error(s_got, s_ref, 2, &worst) == MPSVD_OK && worst == 0.5);
  s_ref[1] = 0.0;
  CHECK(mpsvd_max_rel_sv_error(s_got, s_ref, 2, &worst) == MPSVD_ERR_INVALID_ARGUMENT);
}

static void no_device(void) {
  const double d[2] = {5.0, 3.0};
  mpsvd_matrix* a = stacked_diag(4, d, 2);
  mpsvd_svd_result* r = NULL;
  CHECK(mpsvd_thin_svd(a, MPSVD_EIG_TWOSIDED_JACOBI, 1, &r) == MPSVD_ERR_INTERNAL);
  CHECK(strstr(mpsvd_last_error_message(), "CUDA") != NULL);
  /* argument validation still comes first */
  CHECK(mpsvd_thin_svd(a, MPSVD_EIG_TWOSIDED_JACOBI, 0, &r) == MPSVD_ERR_INVALID_ARGUMENT);
  mpsvd_matrix_destroy(a);
}

static void thin_svd_surface(void) {
  const double d[2] = {5.0, 3.0};
  mpsvd_matrix* a = stacked_diag(4, d, 2);
  mpsvd_svd_result* r = NULL;
  CHECK(mpsvd_thin_svd(a, MPSVD_EIG_TWOSIDED_JACOBI, 1, &r) == MPSVD_OK);
  if (!r) {
    ++g_fail;
    return;
  }
  int64_t count = 0;
  const double* sigma = mpsvd_svd_sigma(r, &count);
  CHECK(count == 2 && sigma[0] == 5.0 && sigma[1] == 3.0);
  const mpsvd_matrix* u = mpsvd_svd_u(r);
  const mpsvd_matrix* vv = mpsvd_svd_v(r);
  CHECK(mpsvd_matrix_rows(u) == 4 && mpsvd_matrix_cols(u) == 2);
  CHECK(mpsvd_matrix_rows(vv) == 2 && mpsvd_matrix_cols(vv) == 2);
  CHECK(mpsvd_matrix_precision(u) == MPSVD_PRECISION_WORKING);
  for (int64_t j = 0; j < 2; ++j)
    for (int64_t i = 0; i < 2; ++i) CHECK(get(vv, i, j) == (i == j ? 1.0 : 0.0));
  for (int64_t j = 0; j < 2; ++j)
    for (int64_t i = 0; i < 4; ++i) CHECK(get(u, i, j) == (i == j ? 1.0 : 0.0));
  CHECK(mpsvd_svd_sync_events(r) == 1);
  CHECK(mpsvd_svd_gram_blocks(r) == 4); /* min(16, m) logical blocks, thinsvd.cpp:66 */
  CHECK(mpsvd_svd_is_qr_baseline(r) == 0);
  double orth = 1.0;
  CHECK(mpsvd_orth_error(u, &orth) == MPSVD_OK && orth <= 16 * 0x1p-24);
  double t[5];
  mpsvd_svd_times(r, t);
  for (int i = 0; i < 4; ++i) CHECK(t[i] >= 0.0);
  CHECK(fabs(t[0] + t[1] + t[2] + t[3] - t[4]) <= 1e-9 + 1e-6 * t[4]);
  mpsvd_svd_destroy(r);

  CHECK(mpsvd_thin_svd(a, (mpsvd_eigensolver)9, 1, &r) == MPSVD_ERR_INVALID_ARGUMENT);
  CHECK(mpsvd_thin_svd(a, MPSVD_EIG_TWOSIDED_JACOBI, 0, &r) == MPSVD_ERR_INVALID_ARGUMENT);
  mpsvd_matrix_destroy(a);

  /* 16 logical blocks from m >= 16; every eigensolver branch; bits do not
   * depend on the thread count (proj/include/mpsvd.h:101-103) */
  mpsvd_matrix* g = NULL;
  const int64_t m = 4096, n = 24;
  CHECK(mpsvd_matrix_create(m, n, MPSVD_PRECISION_WORKING, &g) == MPSVD_OK);
  uint64_t st = 0x9E3779B97F4A7C15ull;  /* full-rank pseudo-random entries in [-1, 1), graded columns */
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      st = st * 6364136223846793005ull + 1442695040888963407ull;
      const double u = (double)(st >> 40) / (double)(1ull << 23) - 1.0;
      CHECK(mpsvd_matrix_set(g, i, j, u * pow(10.0, -3.0 * j / (n - 1))) == MPSVD_OK);
    }
  for (int eig = 0; eig < 3; ++eig) {
    mpsvd_svd_result *r1 = NULL, *r8 = NULL;
    CHECK(mpsvd_thin_svd(g, (mpsvd_eigensolver)eig, 1, &r1) == MPSVD_OK);
    CHECK(mpsvd_thin_svd(g, (mpsvd_eigensolver)eig, 8, &r8) == MPSVD_OK);
    if (!r1 || !r8) continue;
    CHECK(mpsvd_svd_gram_blocks(r1) == 16);
    CHECK(mpsvd_matrix_bitwise_equal(mpsvd_svd_u(r1), mpsvd_svd_u(r8)) == 1);
    CHECK(mpsvd_matrix_bitwise_equal(mpsvd_svd_v(r1), mpsvd_svd_v(r8)) == 1);
    int64_t c1 = 0, c8 = 0;
    const double* s1 = mpsvd_svd_sigma(r1, &c1);
    const double* s8 = mpsvd_svd_sigma(r8, &c8);
    CHECK(c1 == n && c8 == n && memcmp(s1, s8, sizeof(double) * (size_t)n) == 0);
    for (int64_t k = 1; k < n; ++k) CHECK(s1[k] <= s1[k - 1]);
    double bw = 1.0;
    int64_t skipped = -1;
    CHECK(mpsvd_rowwise_backward_error(g, mpsvd_svd_u(r1), s1, c1, mpsvd_svd_v(r1), &bw, &skipped) == MPSVD_OK);
    CHECK(bw <= 100 * sqrt((double)n) * 0x1p-24 && skipped == 0);
    mpsvd_svd_destroy(r1);
    mpsvd_svd_destroy(r8);
  }
  mpsvd_matrix_destroy(g);
}

static void error_payloads(void) {
  /* duplicated column: the Gram matrix has an exactly zero second pivot */
  mpsvd_matrix* a = NULL;
  CHECK(mpsvd_matrix_create(2, 2, MPSVD_PRECISION_WORKING, &a) == MPSVD_OK);
  CHECK(mpsvd_matrix_set(a, 0, 0, 1.0) == MPSVD_OK);
  CHECK(mpsvd_matrix_set(a, 0, 1, 1.0) == MPSVD_OK);
  mpsvd_matrix *q = NULL, *r = NULL;
  CHECK(mpsvd_cholesky_qr(a, &q, &r) == MPSVD_ERR_NOT_POSITIVE_DEFINITE);
  CHECK(mpsvd_last_error_index() == 2);
  CHECK(strlen(mpsvd_last_error_message()) > 0);
  mpsvd_matrix_destroy(a);

  const double d[2] = {1.0, 1e-39};
  mpsvd_matrix* tiny = stacked_diag(2, d, 2);
  mpsvd_svd_result* out = NULL;
  CHECK(mpsvd_thin_svd(tiny, MPSVD_EIG_TWOSIDED_JACOBI, 1, &out) == MPSVD_ERR_TINY_SINGULAR_VALUE);
  CHECK(mpsvd_last_error_index() == 2);
  mpsvd_matrix_destroy(tiny);

  /* a successful call clears the diagnostics */
  const double e[2] = {2.0, 1.0};
  mpsvd_matrix* ok = stacked_diag(3, e, 2);
  CHECK(mpsvd_thin_svd(ok, MPSVD_EIG_TWOSIDED_JACOBI, 1, &out) == MPSVD_OK);
  CHECK(mpsvd_last_error_index() == 0 && strlen(mpsvd_last_error_message()) == 0);
  mpsvd_svd_destroy(out);
  mpsvd_matrix_destroy(ok);
}

int main(int argc, char** argv) {
  const int host_only = argc > 1 && strcmp(argv[1], "--host-only") == 0;
  host_side();
  if (host_only) {
    no_device();
  } else {
    thin_svd_surface();
    error_payloads();
  }
  printf("%s: %d checks, %d failed\n", host_only ? "host-only" : "device", g_checks, g_fail);
  if (g_fail == 0) printf("ALL OK\n");
  return g_fail == 0 ? 0 : 1;
}
