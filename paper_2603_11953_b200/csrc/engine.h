// Host orchestrator interface (engine.cu); used by api.cpp.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "kernels.h"
#include "mpsvd.h"

namespace mpsvd {
namespace engine {

struct Comm;

void check(cudaError_t e, const char* what);
bool device_available();
void comm_unique_id(unsigned char id[128]);
Comm* comm_init(const unsigned char id[128], int nranks, int rank);
void comm_destroy(Comm* c);
std::vector<Comm*> comm_init_all(const std::vector<int>& devs);

class Plan {
 public:
  Plan(long long m_local, long long n, bool f64_working, Comm* comm);
  ~Plan();
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;

  void set_jacobi(double tol, int max_sweeps);
  // spectral branch (thinsvd.cpp:79-105): 0 TwoSidedJacobi, 1 GramCholSvd,
  // 2 OneSidedJacobiOnGram (the last two: binary32 working precision only)
  void set_eigensolver(int choice);
  void ensure_onesided_buffers();
  void ensure_log();
  // Enqueue the whole pipeline on `st` (nullptr: the plan's stream).
  void execute(const void* d_a, long long lda, void* d_u, long long ldu, void* d_sigma, void* d_v,
               cudaStream_t st);
  // host buffers (page-locked) in and out, copies overlapped with the kernels
  void execute_host(const void* h_a, void* d_a, void* h_u, void* d_u, double* h_sigma, double* d_sigma, void* h_v,
                    void* d_v, cudaStream_t st);
  // the kernel sequence of execute (captured into graph_exec)
  void enqueue(const void* d_a, long long lda, void* d_u, long long ldu, void* d_sigma, void* d_v,
               cudaStream_t st);
  mpsvd_exec_info wait();
  // status word handling around hand-assembled stage sequences
  void reset_status(cudaStream_t st);
  void fetch_status(cudaStream_t st);

  // stages (used by execute and by the stage-level entry points)
  void gram(const void* d_a, long long lda, cudaStream_t st);
  // double-double Gram kernels of splits [sb, sb + cnt) (K2z Ozaki or K2 Dot2)
  void gram_dd_splits(const void* d_a, long long lda, int sb, int cnt, cudaStream_t st);
  // multi-rank: the partial Grams (d_mloc) of every rank -> d_m
  void exchange(cudaStream_t st);
  // ||Q^T Q - I||_F in binary64 of a device-resident m_local x n Q in the
  // plan's precision (the plan's Gram stage, exchange included: global over
  // ranks); overwrites the plan's Gram. Synchronous on st.
  double orth_error(const void* d_q, long long ldq, cudaStream_t st);
  void eigen(cudaStream_t st);
  // mixed-precision Cholesky QR (thinsvd.cpp:125-154): Gram (K1), chol (K8),
  // row solves (K10). Q: m x n binary32 (ldq), R: the plan's d_x32 (n x n)
  void cholqr(const void* d_a, long long lda, void* d_q, long long ldq, cudaStream_t st);
  // sort / sign / sigma / V in working precision / W = V Sigma^-1
  void finish(double* sigma, void* v_work, cudaStream_t st);
  double effective_tol() const;

  long long m, n;
  bool dd;
  Comm* comm;
  int device = 0, sm_count = 148;
  double tol = 0.0;
  int max_sweeps = 30;
  int eig_choice = 0;
  int log_sweeps = 0;  // sweeps the rotation log (jws.log) can hold; grown by set_jacobi

  std::vector<int2> tiles;
  std::vector<int> tp_order;  // diagonal tile pairs first (ndiag of them), then the rest
  int ndiag = 0;
  std::vector<longlong2> splits;
  std::vector<int> block_split_begin;
  int ntp = 0, nblocks = 0;
  // K2z (double-double Gram on the int8 tensor cores); MPSVD_DD_GRAM=dot2 selects K2
  bool ozaki = false;
  bool f64_allreduce = false;  // MPSVD_F64_EXCHANGE=allreduce (multi-rank fp64 exchange)
  // K1z (binary32 Gram on the int8 tensor cores, gram_ozaki32.cu): one range
  // launch per logical row block, chunk bounds oz32_bounds[b] .. [b + 1]
  bool oz32 = false;
  int gram_kernel = -1, av_kernel = -1;  // kernels of the last execute (mpsvd_exec_info)
  int oz32_pairs = 0;
  std::vector<long long> oz32_bounds;
  double2* d_oz32_part = nullptr;
  int* d_oz32_bad = nullptr;
  bool oz32_usable(const void* d_a, long long lda) const;
  std::vector<int2> oz_tiles;
  std::vector<int> scb;  // split s = 32-row chunks [scb[s], scb[s + 1])
  int2* d_oz_tiles = nullptr;
  int* d_scb = nullptr;
  int* d_bsb_oz = nullptr;  // block_split_begin x ozaki_groups()
  int* d_oz_e = nullptr;    // column exponents per split
  unsigned char* d_digits = nullptr;

  int2* d_tiles = nullptr;
  int* d_tp_order = nullptr;
  longlong2* d_splits = nullptr;
  int* d_bsb = nullptr;
  double* d_partials = nullptr;
  double* d_bsums = nullptr;   // per-logical-block sums (combine pass 1)
  double* d_m = nullptr;       // n x n higher precision (f64 or dd as double2)
  double* d_mloc = nullptr;    // rank-local partial (N > 1)
  double* d_gather = nullptr;  // all-gathered partials (dd, N > 1)
  dev::JacobiWorkspace jws{};
  int* d_perm = nullptr;
  double *d_lam_hi = nullptr, *d_lam_lo = nullptr, *d_sigma_tmp = nullptr;
  double* d_w = nullptr;
  double* d_vwork_tmp = nullptr;
  void* d_wplanes = nullptr;  // K7 tensor-core W pieces (f32, n <= 128)
  // one-sided branches (onesided.cu), allocated by set_eigensolver
  double* d_r64 = nullptr;      // R = chol(M), binary64
  void* d_x32 = nullptr;        // binary32 R, rotated in place
  double* d_osv = nullptr;      // V scratch of the one-sided solver
  double* d_sigraw = nullptr;   // column norms after convergence
  unsigned long long* d_osaux = nullptr;  // per-sweep flags of the grid-wide solver
  dev::DevStatus* h_status = nullptr;
  cudaStream_t own_stream = nullptr, last_stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int launches = 0;
  bool events_recorded = false;
  struct GraphKey {
    const void* a;
    long long lda;
    void* u;
    long long ldu;
    void* sigma;
    void* v;
    bool operator==(const GraphKey& o) const {
      return a == o.a && lda == o.lda && u == o.u && ldu == o.ldu && sigma == o.sigma && v == o.v;
    }
  };
  cudaStream_t copy_stream = nullptr;  // execute_host's copy engine stream
  cudaEvent_t cev[16] = {}, uev[16] = {}, cdone = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  GraphKey graph_key{};
  int graph_launches = 0;
  bool graph_failed = false;
  std::vector<void*> owned;
};

}  // namespace engine
}  // namespace mpsvd
