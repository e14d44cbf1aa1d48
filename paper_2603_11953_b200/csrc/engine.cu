// Host orchestrator of the B200 thin SVD (host code; compiled by nvcc only
// because it includes the device status layout).
//
// One Plan = every device workspace for one (rows, cols, precision, rank),
// so executing the pipeline allocates nothing:
//
//   K1/K2 gram (split-K over rows, 16 logical blocks x S splits)
//     -> gram_combine (splits in order, blocks along the reference tree)
//     -> [N > 1: NCCL all-gather of the rank partials + the reference tree
//         over ranks (fp64 adds / dd_add), Plan::exchange]
//     -> K4/K5 jacobi (persistent, one barrier per round)
//     -> jacobi_replay (V) -> finish (sort, sign, sigma, V, W = V / sigma)
//     -> K7 av (U = A W)
//
// all on one stream, with CUDA events between the phases for PhaseTimes.
// NCCL is resolved with dlopen on first multi-rank use, so the library loads
// (and its single-GPU path runs) without it.
#include <dlfcn.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "engine.h"
#include "kernels.h"

namespace mpsvd {
namespace engine {

using dev::DevStatus;

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

bool device_available() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return count > 0;
}

// ---------------------------------------------------------------------------
// NCCL through dlopen (minimal ABI subset; types from nccl.h 2.x).
namespace nccl {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
enum { ncclSuccess = 0 };
enum { ncclFloat64 = 8 };
enum { ncclSum = 0 };
struct Api {
  int (*GetUniqueId)(ncclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
};
Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    a.GetUniqueId = (int (*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (int (*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(h, "ncclCommInitRank");
    a.CommInitAll = (int (*)(ncclComm_t*, int, const int*))dlsym(h, "ncclCommInitAll");
    a.AllReduce = (int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
    a.AllGather = (int (*)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllGather");
    a.CommDestroy = (int (*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
    a.GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllReduce && a.AllGather && a.CommDestroy;
  });
  return a;
}
void check(int r, const char* what) {
  if (r != ncclSuccess) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    throw std::runtime_error(std::string("NCCL ") + what + ": " + s);
  }
}
}  // namespace nccl

struct Comm {
  nccl::ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

void comm_unique_id(unsigned char id[128]) {
  auto& a = nccl::api();
  if (!a.ok) throw std::runtime_error("NCCL (libnccl.so.2) not loadable");
  nccl::ncclUniqueId u;
  nccl::check(a.GetUniqueId(&u), "GetUniqueId");
  std::memcpy(id, u.internal, 128);
}

Comm* comm_init(const unsigned char id[128], int nranks, int rank) {
  auto& a = nccl::api();
  if (!a.ok) throw std::runtime_error("NCCL (libnccl.so.2) not loadable");
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank/nranks");
  nccl::ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  auto* c = new Comm;
  c->nranks = nranks;
  c->rank = rank;
  nccl::check(a.CommInitRank(&c->comm, nranks, u, rank), "CommInitRank");
  return c;
}

// One communicator per device of `devs`, all in this process (the
// single-process multi-GPU path of the host-buffer API: one host thread per
// GPU drives its rank).
std::vector<Comm*> comm_init_all(const std::vector<int>& devs) {
  auto& a = nccl::api();
  if (!a.ok || !a.CommInitAll) throw std::runtime_error("NCCL (libnccl.so.2) not loadable");
  const int nd = (int)devs.size();
  std::vector<nccl::ncclComm_t> raw(nd, nullptr);
  nccl::check(a.CommInitAll(raw.data(), nd, devs.data()), "CommInitAll");
  std::vector<Comm*> out(nd);
  for (int r = 0; r < nd; ++r) {
    out[r] = new Comm;
    out[r]->comm = raw[r];
    out[r]->nranks = nd;
    out[r]->rank = r;
  }
  return out;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->comm && nccl::api().CommDestroy) nccl::api().CommDestroy(c->comm);
  delete c;
}

// ---------------------------------------------------------------------------
// Gram schedule: logical blocks over the local rows (reference plan,
// parallel_gram.cpp:57-77, 16 blocks as thinsvd.cpp:66), each cut into
// S splits sized so (tile pairs x splits) fills one wave of resident CTAs.
static void build_schedule(Plan& p) {
  const long long m = p.m, n = p.n;
  const int T = (int)((n + 63) / 64);
  p.tiles.clear();
  p.tp_order.clear();
  for (int ti = 0; ti < T; ++ti)
    for (int tj = ti; tj < T; ++tj) p.tiles.push_back(make_int2(ti, tj));
  p.ntp = (int)p.tiles.size();
  // K1 launches the diagonal tiles and the off-diagonal tiles separately
  for (int tp = 0; tp < p.ntp; ++tp)
    if (p.tiles[tp].x == p.tiles[tp].y) p.tp_order.push_back(tp);
  p.ndiag = (int)p.tp_order.size();
  for (int tp = 0; tp < p.ntp; ++tp)
    if (p.tiles[tp].x != p.tiles[tp].y) p.tp_order.push_back(tp);
  p.nblocks = (int)(m < 16 ? m : 16);
  p.splits.clear();
  p.block_split_begin.assign(1, 0);
  if (p.nblocks == 0) return;
  // Row splits per logical block. Every launch runs a whole number of
  // waves as far as possible: a 2nd wave holding a few CTAs doubles a
  // launch's time (C3: 160 CTAs on 148 SMs). Pick per_block (splits per
  // block) minimising  rows_per_split x sum_launch(waves x cost_per_row),
  // with kernels at 1 CTA/SM (dd), 4/SM (f32 diagonal tiles: 36 DMMA blocks
  // per k-step) and 2/SM (f32 off-diagonal tiles: 64 blocks).
  const long long max_pb = std::max(1LL, (m / p.nblocks + 31) / 32);
  int per_block = 1;
  if (p.ozaki) {
    // K2z: tiles x 6 weight groups x splits CTAs of unequal length (21 ... 1
    // products per chunk); at least 4 waves so the block scheduler evens them out
    dev::ozaki_tiles((int)n, p.oz_tiles);
    const long long per_split = (long long)p.oz_tiles.size() * dev::ozaki_groups();
    const long long slot_bytes = (long long)p.ntp * 64 * 64 * 16 * dev::ozaki_groups();
    while (per_block < 64 && per_block < max_pb && per_split * p.nblocks * per_block < 4LL * p.sm_count &&
           (long long)p.nblocks * (per_block + 1) * slot_bytes <= (1536LL << 20))
      ++per_block;
  }
  double best = 1e300;
  const long long tile_bytes = 64LL * 64 * 8 * (p.dd ? 2 : 1);
  for (int pb = 1; pb <= 64 && pb <= max_pb && !p.ozaki; ++pb) {
    const long long S = (long long)pb * p.nblocks;
    if (pb > 1 && S * p.ntp * tile_bytes > (512LL << 20)) break;  // partial-tile workspace cap
    double cost;
    if (p.dd) {
      const long long waves = (p.ntp * S + p.sm_count - 1) / p.sm_count;
      cost = (double)waves / (double)S;
    } else {
      const int noff = p.ntp - p.ndiag;
      const long long wd = (p.ndiag * S + 4LL * p.sm_count - 1) / (4LL * p.sm_count);
      const long long wo = noff ? (noff * S + 2LL * p.sm_count - 1) / (2LL * p.sm_count) : 0;
      cost = (9.0 * (double)wd + 32.0 * (double)wo) / (double)S;
    }
    if (cost < best * 0.999) {  // prefer fewer splits on ties (smaller combine)
      best = cost;
      per_block = pb;
    }
  }
  const long long base = m / p.nblocks, extra = m % p.nblocks;
  long long row = 0;
  for (int b = 0; b < p.nblocks; ++b) {
    const long long len = base + (b < extra ? 1 : 0);
    long long s = per_block;
    const long long max_s = (len + 31) / 32;
    if (s > max_s) s = max_s;
    if (s < 1) s = 1;
    // piece length rounded up to whole 32-row chunks
    long long piece = (len + s - 1) / s;
    piece = (piece + 31) / 32 * 32;
    for (long long r = row; r < row + len; r += piece) {
      longlong2 sp;
      sp.x = r;
      sp.y = r + piece < row + len ? r + piece : row + len;
      p.splits.push_back(sp);
    }
    p.block_split_begin.push_back((int)p.splits.size());
    row += len;
  }
  if (p.ozaki) {
    // K2z splits are whole 32-row chunks: split starts rounded down
    const long long nch = (m + 31) / 32;
    p.scb.resize(p.splits.size() + 1);
    for (size_t i = 0; i < p.splits.size(); ++i) p.scb[i] = (int)(p.splits[i].x / 32);
    p.scb[p.splits.size()] = (int)nch;
  }
}

template <typename T>
static T* dalloc(size_t count, std::vector<void*>& owned) {
  void* ptr = nullptr;
  if (count == 0) count = 1;
  check(cudaMalloc(&ptr, count * sizeof(T)), "cudaMalloc");
  owned.push_back(ptr);
  return static_cast<T*>(ptr);
}

Plan::Plan(long long m_local, long long n_cols, bool f64_working, Comm* c)
    : m(m_local), n(n_cols), dd(f64_working), comm(c) {
  if (n < 1 || m < 0) throw std::invalid_argument("plan: need n >= 1, m >= 0");
  if (!device_available()) throw std::runtime_error("no CUDA device available");
  check(cudaGetDevice(&device), "cudaGetDevice");
  check(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device), "sm count");
  max_sweeps = dd ? 100 : 30;  // thinsvd.hpp kDdMaxSweeps / jacobi.hpp:31
  std::string gs;
  if (dd && m > 0) {
    // K2z (int8 Ozaki) from 4096 local rows and 128 columns. Its error is
    // relative to the column maxima, not to |x_ki x_kj| (gram_ozaki.cu
    // header): |dM_ij| <= rows * 2^-82 * 2^(E_i + E_j) in the worst case
    // (aligned spiky columns), about sqrt(rows) * 2^-82 * 2^(E_i + E_j) for
    // random signs - far inside K2's Dot2 bound 4 (m u)^2 ||a_i|| ||a_j|| for
    // data whose columns are not dominated by one entry. Below 128 columns
    // the 128 x 128 MMA tiles and the 11 * m * roundup(n, 256)-byte digit
    // planes are mostly padding, so K2 keeps those shapes.
    // MPSVD_DD_GRAM=dot2|ozaki forces one kernel.
    const char* g = getenv("MPSVD_DD_GRAM");
    gs = g ? g : "";
    ozaki = gs == "ozaki" || (gs != "dot2" && m >= 4096 && n >= 128);
    if (ozaki && gs != "ozaki") {
      // K2z partials: at least 16 splits x sub-groups x the upper 64x64 tile
      // pairs in double-double; keep K2 when that alone passes 8 GB (n > ~3300)
      const long long T64 = (n + 63) / 64;
      const long long slot_bytes = T64 * (T64 + 1) / 2 * 64 * 64 * 16;
      if (16LL * dev::ozaki_groups() * slot_bytes > (8LL << 30)) ozaki = false;
    }
  }
  build_schedule(*this);
  if (!dd && m > 0 && n <= 128) {
    // K1z: binary32 Gram on the int8 tensor cores (gram_ozaki32.cu) for tall
    // matrices with 64 < n <= 128, where its one 128 x 128 tile is not mostly
    // padding; MPSVD_F32_GRAM=dmma|ozaki forces K1 / K1z (n <= 128)
    const char* g32 = getenv("MPSVD_F32_GRAM");
    const std::string s32 = g32 ? g32 : "";
    oz32 = s32 == "ozaki" || (s32 != "dmma" && n > 64 && m >= (1LL << 20));
    if (oz32) {
      const long long nch = (m + 31) / 32;
      const int resident = dev::gram_ozaki32_max_pairs();
      oz32_pairs = (int)std::max(1LL, std::min<long long>(std::min(sm_count / 2, resident > 0 ? resident : sm_count / 2),
                                                          nch / 64));
      oz32_bounds.clear();
      const long long base = m / nblocks, extra = m % nblocks;
      long long row = 0;
      for (int b = 0; b < nblocks; ++b) {
        oz32_bounds.push_back(row / 32);
        row += base + (b < extra ? 1 : 0);
      }
      oz32_bounds.push_back(nch);
    }
  }
  if (ozaki) {
    // The whole K2z footprint (digit planes + per-slot partial tiles + the
    // n x n workspaces) must fit in the free device memory with a margin,
    // checked before anything is allocated, so plan creation never fails
    // half-way; otherwise K2 (Dot2) runs.
    const size_t T64 = (size_t)(n + 63) / 64;
    const size_t partial_bytes = splits.size() * dev::ozaki_groups() * T64 * (T64 + 1) / 2 * 64 * 64 * 16;
    const size_t need = dev::ozaki_digit_bytes(m, (int)n) + partial_bytes + (size_t)n * n * 16 * 8;
    size_t free_b = 0, total_b = 0;
    bool fits = cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && need + (size_t(1) << 30) <= free_b;
    void* ptr = nullptr;
    if (fits && cudaMalloc(&ptr, dev::ozaki_digit_bytes(m, (int)n)) == cudaSuccess) {
      d_digits = static_cast<unsigned char*>(ptr);
      owned.push_back(ptr);
    } else {
      cudaGetLastError();
      if (gs == "ozaki") throw std::runtime_error("MPSVD_DD_GRAM=ozaki: the K2z digit planes do not fit");
      ozaki = false;
      build_schedule(*this);
    }
  }
  const size_t nn = (size_t)n * n;
  const size_t esz = dd ? 2 : 1;  // doubles per element of the higher precision
  const int N = (int)(n + (n & 1)), np = N / 2;

  d_tiles = dalloc<int2>(tiles.size(), owned);
  d_tp_order = dalloc<int>(tp_order.size(), owned);
  check(cudaMemcpy(d_tp_order, tp_order.data(), tp_order.size() * sizeof(int), cudaMemcpyHostToDevice),
        "H2D tile order");
  d_splits = dalloc<longlong2>(splits.size(), owned);
  d_bsb = dalloc<int>(block_split_begin.size(), owned);
  check(cudaMemcpy(d_tiles, tiles.data(), tiles.size() * sizeof(int2), cudaMemcpyHostToDevice), "H2D tiles");
  if (!splits.empty())
    check(cudaMemcpy(d_splits, splits.data(), splits.size() * sizeof(longlong2), cudaMemcpyHostToDevice),
          "H2D splits");
  check(cudaMemcpy(d_bsb, block_split_begin.data(), block_split_begin.size() * sizeof(int),
                   cudaMemcpyHostToDevice),
        "H2D bsb");
  const size_t slots = splits.size() * (ozaki ? dev::ozaki_groups() : 1);
  d_partials = dalloc<double>(slots * tiles.size() * 64 * 64 * esz, owned);
  if (ozaki) {
    d_oz_tiles = dalloc<int2>(oz_tiles.size(), owned);
    check(cudaMemcpy(d_oz_tiles, oz_tiles.data(), oz_tiles.size() * sizeof(int2), cudaMemcpyHostToDevice),
          "H2D ozaki tiles");
    d_scb = dalloc<int>(scb.size(), owned);
    check(cudaMemcpy(d_scb, scb.data(), scb.size() * sizeof(int), cudaMemcpyHostToDevice), "H2D scb");
    std::vector<int> b6(block_split_begin.size());
    for (size_t i = 0; i < b6.size(); ++i) b6[i] = block_split_begin[i] * dev::ozaki_groups();
    d_bsb_oz = dalloc<int>(b6.size(), owned);
    check(cudaMemcpy(d_bsb_oz, b6.data(), b6.size() * sizeof(int), cudaMemcpyHostToDevice), "H2D bsb");
    d_oz_e = dalloc<int>(splits.size() * (size_t)n, owned);
  }
  d_bsums = dalloc<double>((size_t)(nblocks > 0 ? nblocks : 1) * tiles.size() * 64 * 64 * esz, owned);
  if (oz32) {
    d_oz32_part = reinterpret_cast<double2*>(dalloc<unsigned char>(dev::gram_ozaki32_partial_bytes(oz32_pairs), owned));
    d_oz32_bad = dalloc<int>(128, owned);
  }
  d_m = dalloc<double>(nn * esz, owned);
  const int nranks = comm ? comm->nranks : 1;
  if (nranks > 1) {
    if (nranks > 16) throw std::invalid_argument("plan: at most 16 ranks (the rank combine tree holds 16 slots)");
    const char* ex = getenv("MPSVD_F64_EXCHANGE");
    f64_allreduce = !dd && ex && std::string(ex) == "allreduce";
    d_mloc = dalloc<double>(nn * esz, owned);
    if (!f64_allreduce) d_gather = dalloc<double>(nn * esz * nranks, owned);
  }
  jws.a = d_m;
  jws.diagbuf = dalloc<double>((size_t)2 * np * 3 * esz + 2, owned);  // + sweep flags
  jws.log = nullptr;  // sized on first set_jacobi / execute for the requested sweep cap
  jws.v = dalloc<double>(nn * esz, owned);
  jws.status = dalloc<DevStatus>(1, owned);
  d_perm = dalloc<int>(n, owned);
  d_lam_hi = dalloc<double>(n, owned);
  d_lam_lo = dalloc<double>(n, owned);
  d_sigma_tmp = dalloc<double>(n, owned);
  d_w = dalloc<double>((size_t)n * dev::av_ldw((int)n), owned);  // W^T, working precision
  check(cudaMemset(d_w, 0, (size_t)n * dev::av_ldw((int)n) * sizeof(double)), "memset W");
  d_vwork_tmp = dalloc<double>(nn, owned);
  // K7 on the tensor cores (f32, n <= 128); MPSVD_AV_SIMT=1 keeps the SIMT kernel
  const char* simt = getenv("MPSVD_AV_SIMT");
  if (!dd && n <= 128 && !(simt && simt[0] == '1'))
    d_wplanes = dalloc<unsigned char>(dev::av_tc_wplanes_bytes((int)n), owned);
  check(cudaMallocHost(&h_status, sizeof(DevStatus)), "cudaMallocHost status");
  check(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking), "stream");
  for (auto& e : ev) check(cudaEventCreate(&e), "event");
}

Plan::~Plan() {
  if (graph_exec) cudaGraphExecDestroy(graph_exec);
  for (auto& e : cev)
    if (e) cudaEventDestroy(e);
  for (auto& e : uev)
    if (e) cudaEventDestroy(e);
  if (cdone) cudaEventDestroy(cdone);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  if (own_stream) cudaStreamDestroy(own_stream);
  if (h_status) cudaFreeHost(h_status);
  for (void* p : owned)
    if (p) cudaFree(p);
}

void Plan::set_jacobi(double t, int sweeps) {
  if (sweeps < 1) throw std::invalid_argument("max_sweeps must be >= 1");
  if (sweeps > 1000) throw std::invalid_argument("max_sweeps must be <= 1000");
  if (t != tol || sweeps != max_sweeps) {  // the captured graph holds the old kernel arguments
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    graph_exec = nullptr;
  }
  tol = t;
  max_sweeps = sweeps;
  ensure_log();
}

// The rotation log holds every sweep's (c, s) pairs for the V replay, so its
// size follows the sweep cap: reallocated (never shrunk) when a larger cap is
// requested.
void Plan::ensure_log() {
  if (max_sweeps <= log_sweeps) return;
  if (graph_exec) {  // the captured graph holds the old log pointer
    cudaGraphExecDestroy(graph_exec);
    graph_exec = nullptr;
  }
  if (jws.log) {
    check(cudaDeviceSynchronize(), "sync before log resize");
    for (auto& p : owned)
      if (p == jws.log) p = nullptr;
    check(cudaFree(jws.log), "free log");
  }
  jws.log = dalloc<double>(dev::jacobi_log_elems((int)n, max_sweeps) * (dd ? 2 : 1), owned);
  log_sweeps = max_sweeps;
}

// Phase events: plain records, or external event nodes while the pipeline
// is being captured into a graph (so they still time the replayed graph).
static void record_event(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  check(cudaStreamIsCapturing(st, &cs), "capture status");
  if (cs == cudaStreamCaptureStatusActive)
    check(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal), "event");
  else
    check(cudaEventRecord(e, st), "event");
}

void Plan::set_eigensolver(int choice) {
  if (choice < 0 || choice > 2) throw std::invalid_argument("unknown eigensolver choice");
  if (choice != 0 && dd) throw std::invalid_argument("the one-sided branches take a binary32 working matrix");
  if (choice == eig_choice) return;
  if (graph_exec) {  // the captured graph holds the other branch's kernels
    cudaGraphExecDestroy(graph_exec);
    graph_exec = nullptr;
  }
  eig_choice = choice;
  if (choice != 0) ensure_onesided_buffers();
}

void Plan::ensure_onesided_buffers() {
  if (d_osv) return;
  const size_t nn = (size_t)n * n;
  d_r64 = dalloc<double>(nn, owned);
  d_x32 = dalloc<float>(nn, owned);
  d_osv = dalloc<double>(nn, owned);
  d_sigraw = dalloc<double>(n, owned);
  d_osaux = dalloc<unsigned long long>(dev::onesided_aux_words(1000), owned);
}

void Plan::cholqr(const void* d_a, long long lda, void* d_q, long long ldq, cudaStream_t st) {
  if (dd) throw std::invalid_argument("cholesky QR takes a binary32 working matrix");
  ensure_onesided_buffers();
  last_stream = st;
  launches = 0;
  check(cudaMemsetAsync(jws.status, 0, sizeof(DevStatus), st), "status reset");
  record_event(ev[0], st);
  gram(d_a, lda, st);
  record_event(ev[1], st);
  check(dev::launch_chol_upper(d_m, (int)n, d_r64, (float*)d_x32, jws.status, st), "chol_upper");
  record_event(ev[2], st);
  check(dev::launch_cholqr_rows((const float*)d_a, lda, m, (int)n, (const float*)d_x32, (float*)d_q, ldq, jws.status,
                                sm_count, st),
        "cholqr_rows");
  launches += 2;
  record_event(ev[3], st);
  events_recorded = true;
  check(cudaMemcpyAsync(h_status, jws.status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st), "status D2H");
}

double Plan::effective_tol() const {
  if (tol > 0.0) return tol;
  return (double)n * (dd ? 0x1p-104 : 0x1p-53);  // jacobi.cpp:274-275; u_dd = 2^-104
}

bool Plan::oz32_usable(const void* d_a, long long lda) const {
  return oz32 && dev::gram_ozaki32_supported((const float*)d_a, lda, m, (int)n);
}

void Plan::gram(const void* d_a, long long lda, cudaStream_t st) {
  const int nranks = comm ? comm->nranks : 1;
  void* target = nranks > 1 ? d_mloc : d_m;
  if (nblocks == 0) {
    check(cudaMemsetAsync(target, 0, (size_t)n * n * sizeof(double) * (dd ? 2 : 1), st), "memset M");
  } else if (oz32_usable(d_a, lda)) {
    // K1z: the same per-logical-block range launches as execute_host
    gram_kernel = 1;
    check(dev::launch_gram_ozaki32_begin(d_oz32_bad, st), "ozaki32 begin");
    for (int b = 0; b < nblocks; ++b)
      check(dev::launch_gram_ozaki32_range((const float*)d_a, lda, m, (int)n, oz32_bounds[b], oz32_bounds[b + 1],
                                           oz32_pairs, d_oz32_part, d_oz32_bad, b > 0, st),
            "gram_ozaki32");
    check(dev::launch_gram_ozaki32_combine(d_oz32_part, oz32_pairs, (int)n, d_oz32_bad, (double*)target, st),
          "gram_ozaki32 combine");
    launches += nblocks + 1;
  } else if (dd) {
    gram_kernel = ozaki ? 3 : 2;
    gram_dd_splits(d_a, lda, 0, (int)splits.size(), st);
    check(dev::launch_gram_combine_dd((const double2*)d_partials, ntp, (int)n, ozaki ? d_bsb_oz : d_bsb, nblocks,
                                      (double2*)d_bsums, (double2*)target, st),
          "gram_combine_dd");
    launches += 2;
  } else {
    gram_kernel = 0;
    check(dev::launch_gram_f32((const float*)d_a, lda, (int)n, d_tiles, ntp, d_tp_order, ndiag,
                               d_tp_order + ndiag, ntp - ndiag, d_splits, (int)splits.size(), (double*)d_partials,
                               st),
          "gram_f32");
    check(dev::launch_gram_combine_f64((const double*)d_partials, ntp, (int)n, d_bsb, nblocks,
                                       (double*)d_bsums, (double*)target, st),
          "gram_combine_f64");
    launches += 2 + (ndiag > 0 ? 1 : 0) + (ntp > ndiag ? 1 : 0);
  }
  if (nranks > 1) exchange(st);
  // K7's column scales need ||a_k||^2 after the eigensolver has overwritten M
  if (d_wplanes) {
    check(dev::launch_av_tc_save_diag((const double*)d_m, (int)n, d_wplanes, st), "save Gram diagonal");
    launches += 1;
  }
}

// The one exchange of the multi-GPU path (north_star (4); the reference's
// join of the per-thread partials, parallel_gram.cpp:93-102). Every rank's
// n x n partial is all-gathered and the ranks' partials are added along the
// reference's fixed tree (0,1),(2,3),... then doubling widths - with dd_add
// for double-double (a plain NCCL sum would drop the lo words), with fp64
// adds otherwise. The combine is our own kernel, so every rank computes the
// same bits by construction, independent of NCCL's algorithm choice, and
// the sum of exactly symmetric partials stays exactly symmetric. At these
// sizes (C4: 128 KiB per rank) the gather is latency-bound like an
// all-reduce. MPSVD_F64_EXCHANGE=allreduce selects an NCCL all-reduce (sum)
// plus a re-mirroring of the upper triangle for fp64 instead.
void Plan::exchange(cudaStream_t st) {
  auto& a = nccl::api();
  const size_t nn = (size_t)n * n;
  if (f64_allreduce) {
    nccl::check(a.AllReduce(d_mloc, d_m, nn, nccl::ncclFloat64, nccl::ncclSum, comm->comm, st), "AllReduce");
    check(dev::launch_mirror_upper((double*)d_m, (int)n, st), "mirror");
  } else {
    nccl::check(a.AllGather(d_mloc, d_gather, nn * (dd ? 2 : 1), nccl::ncclFloat64, comm->comm, st), "AllGather");
    check(dev::launch_block_tree(d_gather, comm->nranks, (int)n, d_m, dd, st), "rank combine");
  }
  launches += 1;
}

double Plan::orth_error(const void* d_q, long long ldq, cudaStream_t st) {
  if (!st) st = own_stream;
  last_stream = st;
  events_recorded = false;
  gram(d_q, ldq, st);
  const size_t nn = (size_t)n * n;
  std::vector<double> g(nn * (dd ? 2 : 1));
  check(cudaMemcpyAsync(g.data(), d_m, g.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H Gram");
  check(cudaStreamSynchronize(st), "orth sync");
  // ||Q^T Q - I||_F over the exactly symmetric Gram (dense.cpp:250-272:
  // binary64); the double-double Gram contributes (hi - delta) + lo
  double sum = 0.0;
  for (long long j = 0; j < n; ++j)
    for (long long i = 0; i <= j; ++i) {
      const size_t k = (size_t)j * n + i;
      const double delta = i == j ? 1.0 : 0.0;
      const double d = dd ? (g[2 * k] - delta) + g[2 * k + 1] : g[k] - delta;
      sum += (i == j ? 1.0 : 2.0) * d * d;
    }
  return std::sqrt(sum);
}

void Plan::gram_dd_splits(const void* d_a, long long lda, int sb, int cnt, cudaStream_t st) {
  if (ozaki) {
    check(dev::launch_gram_ozaki((const double*)d_a, lda, m, (int)n, d_scb, scb.data(), (int)splits.size(), sb, cnt,
                                 d_oz_tiles, (int)oz_tiles.size(), d_oz_e, d_digits, (double2*)d_partials, ntp,
                                 sm_count, st),
          "gram_ozaki");
    launches += 3;
  } else {
    check(dev::launch_gram_dd((const double*)d_a, lda, (int)n, d_tiles, ntp, d_splits + sb, cnt,
                              (double2*)d_partials + (size_t)sb * ntp * 64 * 64, st),
          "gram_dd");
    launches += 1;
  }
}

void Plan::eigen(cudaStream_t st) {
  if (eig_choice == 1) {  // GramCholSvd: chol in binary64, one-sided Jacobi of fl32(R)
    check(dev::launch_chol_upper(d_m, (int)n, d_r64, (float*)d_x32, jws.status, st), "chol_upper");
    check(dev::launch_onesided(true, d_x32, d_osv, (int)n, (int)n, tol > 0.0 ? tol : (double)n * 0x1p-24, max_sweeps,
                               jws.status, d_sigraw, (double*)jws.v, d_osaux, sm_count, st),
          "onesided f32");
    launches += 2;
    return;
  }
  if (eig_choice == 2) {  // OneSidedJacobiOnGram: one-sided Jacobi of M in binary64 (M rotated in place)
    check(dev::launch_onesided(false, d_m, d_osv, (int)n, (int)n, tol > 0.0 ? tol : (double)n * 0x1p-53, max_sweeps,
                               jws.status, d_sigraw, (double*)jws.v, d_osaux, sm_count, st),
          "onesided f64");
    launches += 1;
    return;
  }
  ensure_log();
  bool fused = false;
  check(dev::launch_jacobi(dd, (int)n, effective_tol(), max_sweeps, jws, sm_count, st, &fused), "jacobi");
  launches += 1;
  if (!fused) {
    check(dev::launch_jacobi_replay(dd, (int)n, jws, st), "jacobi_replay");
    launches += 1;
  }
}

// The pipeline is captured once per set of device pointers into a CUDA graph
// and replayed (saves the per-kernel launch gaps; ~9 launches per SVD).
// MPSVD_NO_GRAPH=1 launches the kernels directly; so does any capture error.
void Plan::finish(double* sig, void* vw, cudaStream_t st) {
  if (eig_choice == 0) {
    check(dev::launch_finish(dd, (int)n, jws, d_perm, d_lam_hi, d_lam_lo, sig, vw, d_w, dd ? 1 : 0, st), "finish");
  } else {
    check(dev::launch_onesided_sort(d_sigraw, (int)n, eig_choice == 1 ? 0 : 1, jws.status, d_perm, sig, st),
          "onesided sort");
    check(dev::launch_finish_columns_f64((int)n, (const double*)jws.v, jws.status, d_perm, sig, vw, d_w, 0, st),
          "finish columns");
  }
  launches += 2;
}

void Plan::execute(const void* d_a, long long lda, void* d_u, long long ldu, void* d_sigma, void* d_v,
                   cudaStream_t st) {
  if (!st) st = own_stream;
  last_stream = st;
  ensure_log();
  static const bool no_graph = getenv("MPSVD_NO_GRAPH") != nullptr || getenv("MPSVD_JACOBI_TRACE") != nullptr ||
                               getenv("MPSVD_AV_DBG") != nullptr;
  // multi-GPU plans launch directly: a failed capture must never leave a
  // half-recorded NCCL collective behind (and the graph saves only ~15 us)
  if (no_graph || graph_failed || (comm && comm->nranks > 1)) {
    enqueue(d_a, lda, d_u, ldu, d_sigma, d_v, st);
    return;
  }
  const GraphKey key{d_a, lda, d_u, ldu, d_sigma, d_v};
  if (!graph_exec || !(key == graph_key)) {
    if (graph_exec) {
      cudaGraphExecDestroy(graph_exec);
      graph_exec = nullptr;
    }
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(own_stream, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      try {
        enqueue(d_a, lda, d_u, ldu, d_sigma, d_v, own_stream);
      } catch (...) {
        ok = false;
      }
      ok = (cudaStreamEndCapture(own_stream, &g) == cudaSuccess) && ok && g;
    }
    if (ok) ok = cudaGraphInstantiate(&graph_exec, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) {
      cudaGetLastError();  // clear a capture error; run uncaptured from now on
      graph_exec = nullptr;
      graph_failed = true;
      enqueue(d_a, lda, d_u, ldu, d_sigma, d_v, st);
      return;
    }
    graph_key = key;
    graph_launches = launches;
  }
  check(cudaGraphLaunch(graph_exec, st), "graph launch");
  launches = graph_launches;
  events_recorded = true;
}


void Plan::enqueue(const void* d_a, long long lda, void* d_u, long long ldu, void* d_sigma, void* d_v,
                   cudaStream_t st) {
  launches = 0;
  check(cudaMemsetAsync(jws.status, 0, sizeof(DevStatus), st), "status reset");
  record_event(ev[0], st);
  gram(d_a, lda, st);
  record_event(ev[1], st);
  eigen(st);
  double* sig = d_sigma ? (double*)d_sigma : d_sigma_tmp;
  void* vw = d_v ? d_v : d_vwork_tmp;
  finish(sig, vw, st);
  record_event(ev[2], st);
  av_kernel = -1;
  if (d_u && m > 0) {
    av_kernel = dd ? 2 : (d_wplanes && dev::av_tc_supported((const float*)d_a, lda, m, (int)n, ldu)) ? 1 : 0;
    if (dd)
      check(dev::launch_av_dmma_f64((const double*)d_a, lda, m, (int)n, (const double*)d_w, (double*)d_u, ldu,
                                    jws.status, st),
            "av_dmma_f64");
    else if (d_wplanes && dev::av_tc_supported((const float*)d_a, lda, m, (int)n, ldu)) {
      check(dev::launch_av_tc_f32((const float*)d_a, lda, m, (int)n, (const float*)d_w, d_wplanes, (float*)d_u,
                                  ldu, jws.status, sm_count, st),
            "av_tc_f32");
      launches += 1;  // + the W split kernel below
    } else
      check(dev::launch_av_f32((const float*)d_a, lda, m, (int)n, (const float*)d_w, (float*)d_u, ldu,
                               jws.status, st),
            "av_f32");
    launches += 1;
  }
  record_event(ev[3], st);
  events_recorded = true;
  check(cudaMemcpyAsync(h_status, jws.status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st), "status D2H");
}

// Host-buffer pipeline (the C ABI / C++ API path on one GPU). The upload of
// A is cut at the 16 logical row blocks and each block's Gram kernels start
// as soon as its rows have landed (same kernels, splits and partial slots as
// execute(), so the result is bit-identical to it); U is formed in row
// chunks, each downloaded while the next one is computed. The PCIe copies,
// not the kernels, dominate this path (C2: ~10 ms of copies vs 0.57 ms of
// kernels); this hides the Gram and U kernels behind them.
void Plan::execute_host(const void* h_a, void* d_a, void* h_u, void* d_u, double* h_sigma, double* d_sigma, void* h_v,
                        void* d_v, cudaStream_t st) {
  if (comm) throw std::invalid_argument("execute_host: single-GPU plans only");
  ensure_log();
  if (!copy_stream) {
    check(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking), "copy stream");
    for (auto& e : cev) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (auto& e : uev) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    check(cudaEventCreateWithFlags(&cdone, cudaEventDisableTiming), "event");
  }
  cudaStream_t cs = copy_stream;
  last_stream = st;
  launches = 0;
  const size_t elt = dd ? 8 : 4;
  const size_t pitch = (size_t)m * elt;
  const size_t esz = dd ? 2 : 1;
  check(cudaMemsetAsync(jws.status, 0, sizeof(DevStatus), st), "status reset");
  // the copy stream must not overtake work already queued on st
  check(cudaEventRecord(cdone, st), "event");
  check(cudaStreamWaitEvent(cs, cdone, 0), "wait");
  record_event(ev[0], st);
  const bool k1z = oz32_usable(d_a, m);
  gram_kernel = k1z ? 1 : dd ? (ozaki ? 3 : 2) : 0;
  if (k1z) check(dev::launch_gram_ozaki32_begin(d_oz32_bad, st), "ozaki32 begin");
  {
    const long long base = m / nblocks, extra = m % nblocks;
    long long row = 0;
    for (int b = 0; b < nblocks; ++b) {
      const long long len = base + (b < extra ? 1 : 0);
      check(cudaMemcpy2DAsync((char*)d_a + row * elt, pitch, (const char*)h_a + row * elt, pitch, len * elt, n,
                              cudaMemcpyHostToDevice, cs),
            "H2D A block");
      check(cudaEventRecord(cev[b], cs), "event");
      check(cudaStreamWaitEvent(st, cev[b], 0), "wait");
      const int sb = block_split_begin[b], cnt = block_split_begin[b + 1] - sb;
      if (k1z) {
        // K1z range b: its chunks end at or before this block's last row
        check(dev::launch_gram_ozaki32_range((const float*)d_a, m, m, (int)n, oz32_bounds[b], oz32_bounds[b + 1],
                                             oz32_pairs, d_oz32_part, d_oz32_bad, b > 0, st),
              "gram_ozaki32");
        launches += 1;
      } else if (dd) {
        gram_dd_splits(d_a, m, sb, cnt, st);
      } else {
        check(dev::launch_gram_f32((const float*)d_a, m, (int)n, d_tiles, ntp, d_tp_order, ndiag, d_tp_order + ndiag,
                                   ntp - ndiag, d_splits + sb, cnt, d_partials + (size_t)sb * ntp * 64 * 64, st),
              "gram_f32");
        launches += (ndiag > 0 ? 1 : 0) + (ntp > ndiag ? 1 : 0);
      }
      row += len;
    }
  }
  if (k1z)
    check(dev::launch_gram_ozaki32_combine(d_oz32_part, oz32_pairs, (int)n, d_oz32_bad, (double*)d_m, st),
          "gram_ozaki32 combine");
  else if (dd)
    check(dev::launch_gram_combine_dd((const double2*)d_partials, ntp, (int)n, ozaki ? d_bsb_oz : d_bsb, nblocks,
                                      (double2*)d_bsums, (double2*)d_m, st),
          "gram_combine_dd");
  else
    check(dev::launch_gram_combine_f64((const double*)d_partials, ntp, (int)n, d_bsb, nblocks, (double*)d_bsums,
                                       (double*)d_m, st),
          "gram_combine_f64");
  launches += k1z ? 1 : 2;
  if (d_wplanes) {
    check(dev::launch_av_tc_save_diag((const double*)d_m, (int)n, d_wplanes, st), "save Gram diagonal");
    launches += 1;
  }
  (void)esz;
  record_event(ev[1], st);
  eigen(st);
  finish(d_sigma, d_v, st);
  record_event(ev[2], st);
  // sigma and V travel while U is formed
  check(cudaEventRecord(cdone, st), "event");
  check(cudaStreamWaitEvent(cs, cdone, 0), "wait");
  check(cudaMemcpyAsync(h_sigma, d_sigma, n * sizeof(double), cudaMemcpyDeviceToHost, cs), "D2H sigma");
  check(cudaMemcpyAsync(h_v, d_v, (size_t)n * n * elt, cudaMemcpyDeviceToHost, cs), "D2H V");
  const bool tc = !dd && d_wplanes && dev::av_tc_supported((const float*)d_a, m, m, (int)n, m);
  av_kernel = dd ? 2 : tc ? 1 : 0;
  constexpr int kChunks = 16;
  long long r0 = 0;
  bool first = true;  // the first launched chunk splits W into its pieces
  for (int k = 0; k < kChunks && r0 < m; ++k) {
    long long r1 = (k + 1 == kChunks) ? m : ((long long)(k + 1) * m / kChunks) / 128 * 128;
    if (r1 <= r0) continue;
    const long long rows = r1 - r0;
    if (dd)
      check(dev::launch_av_dmma_f64((const double*)d_a + r0, m, rows, (int)n, (const double*)d_w, (double*)d_u + r0, m,
                                    jws.status, st),
            "av_dmma_f64");
    else if (tc) {
      check(dev::launch_av_tc_f32((const float*)d_a + r0, m, rows, (int)n, (const float*)d_w, d_wplanes,
                                  (float*)d_u + r0, m, jws.status, sm_count, st, first),
            "av_tc_f32");
      if (first) launches += 1;
      first = false;
    } else
      check(dev::launch_av_f32((const float*)d_a + r0, m, rows, (int)n, (const float*)d_w, (float*)d_u + r0, m,
                               jws.status, st),
            "av_f32");
    launches += 1;
    check(cudaEventRecord(uev[k], st), "event");
    check(cudaStreamWaitEvent(cs, uev[k], 0), "wait");
    check(cudaMemcpy2DAsync((char*)h_u + r0 * elt, pitch, (const char*)d_u + r0 * elt, pitch, rows * elt, n,
                            cudaMemcpyDeviceToHost, cs),
          "D2H U chunk");
    r0 = r1;
  }
  record_event(ev[3], st);
  events_recorded = true;
  check(cudaMemcpyAsync(h_status, jws.status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st), "status D2H");
  // join: wait() synchronises st, which now also covers the copy stream
  check(cudaEventRecord(cdone, cs), "event");
  check(cudaStreamWaitEvent(st, cdone, 0), "wait");
}

void Plan::reset_status(cudaStream_t st) {
  last_stream = st;
  events_recorded = false;
  check(cudaMemsetAsync(jws.status, 0, sizeof(DevStatus), st), "status reset");
}

void Plan::fetch_status(cudaStream_t st) {
  check(cudaMemcpyAsync(h_status, jws.status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st), "status D2H");
}

mpsvd_exec_info Plan::wait() {
  check(cudaStreamSynchronize(last_stream ? last_stream : own_stream), "stream sync");
  mpsvd_exec_info info;
  std::memset(&info, 0, sizeof(info));
  info.status = h_status->status;
  info.error_index = h_status->index;
  info.error_value = h_status->value;
  info.sweeps = h_status->sweeps;
  info.rotations = h_status->rotations;
  info.rounds = h_status->rounds;
  if (events_recorded) {
    float ms = 0;
    check(cudaEventElapsedTime(&ms, ev[0], ev[1]), "event time");
    info.ms_gram = ms;
    check(cudaEventElapsedTime(&ms, ev[1], ev[2]), "event time");
    info.ms_eigen = ms;
    check(cudaEventElapsedTime(&ms, ev[2], ev[3]), "event time");
    info.ms_compute_u = ms;
  }
  info.kernel_launches = launches;
  info.gram_kernel = gram_kernel;
  info.av_kernel = av_kernel;
  return info;
}

}  // namespace engine
}  // namespace mpsvd
