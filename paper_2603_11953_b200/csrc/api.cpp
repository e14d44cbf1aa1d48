// Public C++ API (include/mpsvd/*.hpp) and C ABI (include/mpsvd.h) of the
// B200 thin SVD. The C ABI wraps the C++ API exactly like the reference's
// capi.cpp wraps its core (proj/src/capi.cpp:50-81,245-252): every entry runs
// inside `guarded`, which maps the exception hierarchy to mpsvd_status codes
// and keeps the message and the 1-based index thread-locally.
//
// The compute entry points run only on the GPU: with no usable CUDA device
// they fail with MPSVD_ERR_INTERNAL ("no CUDA device"); there is no CPU path.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "engine.h"
#include "mpsvd.h"
#include "mpsvd/metrics.hpp"
#include "mpsvd/io.hpp"
#include "mpsvd/thinsvd.hpp"
#include "mpsvd/types.hpp"

namespace mpsvd {

// ---------------------------------------------------------------------------
// errors
NotPositiveDefiniteError::NotPositiveDefiniteError(index_t p, double v)
    : Error("matrix not positive definite at pivot " + std::to_string(p) + " (value " + std::to_string(v) +
            "); condition number too large for chosen higher precision"),
      pivot(p),
      value(v) {}
NoConvergenceError::NoConvergenceError(int s, double w)
    : Error("Jacobi iteration did not converge in " + std::to_string(s) +
            " sweeps; final max normalized off-diagonal " + std::to_string(w)),
      sweeps(s),
      max_offdiag(w) {}
ZeroColumnError::ZeroColumnError(index_t c) : Error("column " + std::to_string(c) + " has zero norm"), column(c) {}
ZeroDivisorError::ZeroDivisorError(index_t i) : Error("zero scale entry at index " + std::to_string(i)), index(i) {}
CastOverflowError::CastOverflowError(index_t r, index_t c, double v)
    : Error("entry (" + std::to_string(r) + "," + std::to_string(c) + ") overflows the working precision"),
      row(r),
      col(c),
      value(v) {}
TinySingularValueError::TinySingularValueError(index_t i, double v)
    : Error("singular value " + std::to_string(i) + " = " + std::to_string(v) +
            " underflows the working precision normal range"),
      index(i),
      value(v) {}

// ---------------------------------------------------------------------------
// host buffers: page-locked for sizes worth pinning, plain heap otherwise
namespace detail {
static constexpr std::size_t kPinThreshold = 1u << 20;

// Page-locking is expensive (the driver pins every page), so freed pinned
// blocks are kept in a small size-keyed pool and handed to the next buffer
// of the same size: repeated calls on the same shapes pay it once.
namespace {
struct PinnedPool {
  std::mutex mu;
  std::multimap<std::size_t, void*> free_blocks;
  std::size_t cached = 0;
  static constexpr std::size_t kMaxCached = std::size_t(48) << 30;
  void* take(std::size_t bytes) {
    std::lock_guard<std::mutex> g(mu);
    auto it = free_blocks.find(bytes);
    if (it == free_blocks.end()) return nullptr;
    void* p = it->second;
    free_blocks.erase(it);
    cached -= bytes;
    return p;
  }
  void give(void* p, std::size_t bytes) {
    {
      std::lock_guard<std::mutex> g(mu);
      if (cached + bytes <= kMaxCached) {
        free_blocks.emplace(bytes, p);
        cached += bytes;
        return;
      }
    }
    cudaFreeHost(p);
  }
};
PinnedPool& pool() {
  static PinnedPool* p = new PinnedPool;  // leaked on purpose: outlives static teardown
  return *p;
}
}  // namespace

HostBuffer::HostBuffer(std::size_t bytes, bool zero) : bytes_(bytes) {
  if (bytes == 0) return;
  if (bytes >= kPinThreshold && engine::device_available()) {
    ptr_ = pool().take(bytes);
    if (!ptr_ && cudaMallocHost(&ptr_, bytes) != cudaSuccess) {
      cudaGetLastError();
      ptr_ = nullptr;
    }
    if (ptr_) {
      pinned_ = true;
      if (zero) std::memset(ptr_, 0, bytes);
      return;
    }
  }
  ptr_ = zero ? std::calloc(bytes, 1) : std::malloc(bytes);
  if (!ptr_) throw std::bad_alloc();
}
HostBuffer::HostBuffer(const HostBuffer& o) : HostBuffer(o.bytes_) {
  if (bytes_) std::memcpy(ptr_, o.ptr_, bytes_);
}
HostBuffer& HostBuffer::operator=(const HostBuffer& o) {
  if (this != &o) {
    HostBuffer t(o);
    *this = std::move(t);
  }
  return *this;
}
HostBuffer::HostBuffer(HostBuffer&& o) noexcept : ptr_(o.ptr_), bytes_(o.bytes_), pinned_(o.pinned_) {
  o.ptr_ = nullptr;
  o.bytes_ = 0;
  o.pinned_ = false;
}
HostBuffer& HostBuffer::operator=(HostBuffer&& o) noexcept {
  if (this != &o) {
    release();
    ptr_ = o.ptr_;
    bytes_ = o.bytes_;
    pinned_ = o.pinned_;
    o.ptr_ = nullptr;
    o.bytes_ = 0;
    o.pinned_ = false;
  }
  return *this;
}
HostBuffer::~HostBuffer() { release(); }
void HostBuffer::release() {
  if (!ptr_) return;
  if (pinned_)
    pool().give(ptr_, bytes_);
  else
    std::free(ptr_);
  ptr_ = nullptr;
}
}  // namespace detail

DenseMatrix::DenseMatrix(index_t rows, index_t cols, Precision prec)
    : rows_(rows), cols_(cols), prec_(prec) {
  if (rows < 0 || cols < 0) throw InvalidArgument("negative matrix dimension");
  const std::size_t elt = prec == Precision::Working ? sizeof(float) : sizeof(double);
  buf_ = detail::HostBuffer(static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols) * elt);
}

DenseMatrix DenseMatrix::uninitialized(index_t rows, index_t cols, Precision prec) {
  if (rows < 0 || cols < 0) throw InvalidArgument("negative matrix dimension");
  DenseMatrix a;
  a.rows_ = rows;
  a.cols_ = cols;
  a.prec_ = prec;
  const std::size_t elt = prec == Precision::Working ? sizeof(float) : sizeof(double);
  a.buf_ = detail::HostBuffer(static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols) * elt, false);
  return a;
}

DenseMatrix DenseMatrix::identity(index_t n, Precision prec) {
  DenseMatrix a(n, n, prec);
  for (index_t i = 0; i < n; ++i) a.set(i, i, 1.0);
  return a;
}

double DenseMatrix::get(index_t i, index_t j) const {
  const std::size_t k = static_cast<std::size_t>(j) * rows_ + i;
  return prec_ == Precision::Working ? static_cast<double>(fptr()[k]) : dptr()[k];
}

void DenseMatrix::set(index_t i, index_t j, double v) {
  const std::size_t k = static_cast<std::size_t>(j) * rows_ + i;
  if (prec_ == Precision::Working)
    fptr()[k] = static_cast<float>(v);
  else
    dptr()[k] = v;
}

bool DenseMatrix::bitwise_equal(const DenseMatrix& o) const {
  if (rows_ != o.rows_ || cols_ != o.cols_ || prec_ != o.prec_) return false;
  const std::size_t bytes = static_cast<std::size_t>(size()) * (prec_ == Precision::Working ? 4 : 8);
  return bytes == 0 || std::memcmp(buf_.data(), o.buf_.data(), bytes) == 0;
}

// ---------------------------------------------------------------------------
// Per-thread device resources: calls on distinct threads never share a plan
// or a stream, which keeps mp_thin_svd reentrant.
namespace {

struct Bundle {
  std::unique_ptr<engine::Plan> plan;
  void* d_a = nullptr;
  void* d_u = nullptr;
  double* d_sigma = nullptr;
  void* d_v = nullptr;
  double* h_sigma = nullptr;  // page-locked
  ~Bundle() {
    if (h_sigma) cudaFreeHost(h_sigma);
    cudaFree(d_a);
    cudaFree(d_u);
    cudaFree(d_sigma);
    cudaFree(d_v);
  }
};

using Key = std::tuple<long long, long long, bool>;

Bundle& bundle_for(long long m, long long n, bool f64) {
  thread_local std::map<Key, std::unique_ptr<Bundle>> cache;
  const Key key{m, n, f64};
  auto it = cache.find(key);
  if (it != cache.end()) return *it->second;
  if (cache.size() >= 4) cache.clear();  // bounded: large plans hold GBs
  auto b = std::make_unique<Bundle>();
  b->plan = std::make_unique<engine::Plan>(m, n, f64, nullptr);
  const std::size_t elt = f64 ? 8 : 4;
  engine::check(cudaMalloc(&b->d_a, std::max<std::size_t>(1, m * n * elt)), "cudaMalloc A");
  engine::check(cudaMalloc(&b->d_u, std::max<std::size_t>(1, m * n * elt)), "cudaMalloc U");
  engine::check(cudaMalloc((void**)&b->d_sigma, n * sizeof(double)), "cudaMalloc sigma");
  engine::check(cudaMalloc(&b->d_v, n * n * elt), "cudaMalloc V");
  engine::check(cudaMallocHost((void**)&b->h_sigma, n * sizeof(double)), "cudaMallocHost sigma");
  auto& ref = *b;
  cache.emplace(key, std::move(b));
  return ref;
}

void require_device() {
  if (!engine::device_available()) throw std::runtime_error("no CUDA device: the mpsvd GPU path cannot run");
}

void raise_device_status(const mpsvd_exec_info& info, int max_sweeps) {
  switch (info.status) {
    case 0:
      return;
    case 2:
      throw NotPositiveDefiniteError(info.error_index, info.error_value);
    case 3:
      throw NoConvergenceError(max_sweeps, info.error_value);
    case 7:
      throw TinySingularValueError(info.error_index, info.error_value);
    case 4:
      throw ZeroColumnError(info.error_index);
    case 6:  // the column travels in the sweeps field (no sweep has run)
      throw CastOverflowError(info.error_index, info.sweeps, info.error_value);
    case 1:
      throw InvalidArgument("non-finite entry (" + std::to_string(info.error_index) + "," +
                            std::to_string(info.sweeps) + ") in cast");
    default:
      throw std::runtime_error("device pipeline failed with status " + std::to_string(info.status));
  }
}

using Clock = std::chrono::steady_clock;

// ---------------------------------------------------------------------------
// Single-process multi-GPU path of the host-buffer entry points (SURVEY.md
// §5: one cached NCCL communicator set per process thread, one host thread
// per GPU). Rows of the caller's column-major A are block-sharded across the
// devices (the reference partition rule, parallel_gram.cpp:69-75); every
// device uploads its rows with one strided copy, runs the pipeline with the
// one Gram exchange (Plan::exchange), the redundant Jacobi and its rows of
// U, which go straight back into the caller's U. Device selection:
// MPSVD_DEVICES = "all" (default: every visible device) | a comma-separated
// device list ("0", "0,2,3"); a problem is sharded only when every device gets at least
// MPSVD_SHARD_MIN_ROWS rows (default 2^18: below that the per-device
// launches and copies outweigh the split). MPSVD_SHARD_FORCE=1 takes the
// sharded path even on one device (tests: it must give the single-GPU bits).
std::vector<int> shard_devices(long long m) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1) {
    cudaGetLastError();
    return {};
  }
  std::vector<int> devs;
  const char* env = getenv("MPSVD_DEVICES");
  const std::string s = env ? env : "all";
  if (s.empty() || s == "all") {
    for (int d = 0; d < count; ++d) devs.push_back(d);
  } else {
    if (s.find_first_not_of("0123456789,") != std::string::npos)
      throw InvalidArgument("MPSVD_DEVICES must be \"all\" or a comma-separated device list");
    size_t pos = 0;
    while (pos < s.size()) {
      const size_t e = s.find(',', pos);
      const int d = std::atoi(s.substr(pos, e == std::string::npos ? std::string::npos : e - pos).c_str());
      if (d < 0 || d >= count) throw InvalidArgument("MPSVD_DEVICES names a device that is not visible");
      devs.push_back(d);
      if (e == std::string::npos) break;
      pos = e + 1;
    }
  }
  const char* mr = getenv("MPSVD_SHARD_MIN_ROWS");
  const long long min_rows = mr ? std::max(1LL, std::atoll(mr)) : (1LL << 18);
  while (devs.size() > 1 && m < (long long)devs.size() * min_rows) devs.pop_back();
  return devs;
}

struct ShardSet {
  std::vector<int> devs;
  std::vector<engine::Comm*> comms;
  std::vector<std::unique_ptr<Bundle>> parts;
  std::vector<long long> row0, rows;
  ~ShardSet() {
    for (size_t r = 0; r < parts.size(); ++r) {
      cudaSetDevice(devs[r]);
      parts[r].reset();
    }
    for (auto* c : comms) engine::comm_destroy(c);
  }
};

ShardSet& shard_set_for(const std::vector<int>& devs, long long m, long long n, bool f64) {
  using SKey = std::tuple<std::vector<int>, long long, long long, bool>;
  thread_local std::map<SKey, std::unique_ptr<ShardSet>> cache;
  const SKey key{devs, m, n, f64};
  auto it = cache.find(key);
  if (it != cache.end()) return *it->second;
  if (cache.size() >= 2) cache.clear();  // bounded: every device holds a plan
  int prev = 0;
  cudaGetDevice(&prev);
  auto set = std::make_unique<ShardSet>();
  set->devs = devs;
  set->comms = engine::comm_init_all(devs);
  const int p = (int)devs.size();
  const long long base = m / p, extra = m % p;
  long long row = 0;
  for (int r = 0; r < p; ++r) {
    const long long len = base + (r < extra ? 1 : 0);
    set->row0.push_back(row);
    set->rows.push_back(len);
    row += len;
  }
  set->parts.resize(p);
  std::vector<std::string> errs(p);
  std::vector<std::thread> th;
  for (int r = 0; r < p; ++r)
    th.emplace_back([&, r] {
      try {
        engine::check(cudaSetDevice(devs[r]), "cudaSetDevice");
        auto b = std::make_unique<Bundle>();
        const long long ml = set->rows[r];
        b->plan = std::make_unique<engine::Plan>(ml, n, f64, set->comms[r]);
        const std::size_t elt = f64 ? 8 : 4;
        engine::check(cudaMalloc(&b->d_a, std::max<std::size_t>(1, ml * n * elt)), "cudaMalloc A");
        engine::check(cudaMalloc(&b->d_u, std::max<std::size_t>(1, ml * n * elt)), "cudaMalloc U");
        engine::check(cudaMalloc((void**)&b->d_sigma, n * sizeof(double)), "cudaMalloc sigma");
        engine::check(cudaMalloc(&b->d_v, n * n * elt), "cudaMalloc V");
        engine::check(cudaMallocHost((void**)&b->h_sigma, n * sizeof(double)), "cudaMallocHost sigma");
        set->parts[r] = std::move(b);
      } catch (const std::exception& e) {
        errs[r] = e.what();
      }
    });
  for (auto& t : th) t.join();
  cudaSetDevice(prev);
  for (int r = 0; r < p; ++r)
    if (!errs[r].empty()) throw std::runtime_error("device " + std::to_string(devs[r]) + ": " + errs[r]);
  auto& ref = *set;
  cache.emplace(key, std::move(set));
  return ref;
}

ThinSvdResult run_thin_svd_sharded(const DenseMatrix& a, const JacobiConfig& cfg, bool f64, EigensolverChoice choice,
                                   const std::vector<int>& devs, Clock::time_point t0) {
  const long long m = a.rows(), n = a.cols();
  ShardSet& set = shard_set_for(devs, m, n, f64);
  const int p = (int)devs.size();
  const Precision wp = f64 ? Precision::Higher : Precision::Working;
  ThinSvdResult out;
  out.factors.u = DenseMatrix::uninitialized(m, n, wp);
  out.factors.v = DenseMatrix::uninitialized(n, n, wp);
  out.factors.sigma.assign(n, 0.0);
  out.factors.precision = wp;
  const std::size_t elt = f64 ? 8 : 4;
  const int eig = choice == EigensolverChoice::TwoSidedJacobi ? 0 : choice == EigensolverChoice::GramCholSvd ? 1 : 2;
  std::vector<mpsvd_exec_info> infos(p);
  std::vector<std::string> errs(p);
  std::vector<std::thread> th;
  for (int r = 0; r < p; ++r)
    th.emplace_back([&, r] {
      try {
        engine::check(cudaSetDevice(devs[r]), "cudaSetDevice");
        Bundle& b = *set.parts[r];
        engine::Plan& pl = *b.plan;
        pl.set_jacobi(cfg.tol, cfg.max_sweeps);
        pl.set_eigensolver(eig);
        cudaStream_t st = pl.own_stream;
        const long long ml = set.rows[r], r0 = set.row0[r];
        if (ml > 0)  // this rank's rows of every column: one strided copy
          engine::check(cudaMemcpy2DAsync(b.d_a, ml * elt, (const char*)a.raw() + r0 * elt, m * elt, ml * elt, n,
                                          cudaMemcpyHostToDevice, st),
                        "H2D A rows");
        pl.execute(b.d_a, std::max(1LL, ml), b.d_u, std::max(1LL, ml), b.d_sigma, b.d_v, st);
        if (ml > 0)
          engine::check(cudaMemcpy2DAsync((char*)out.factors.u.raw() + r0 * elt, m * elt, b.d_u, ml * elt, ml * elt, n,
                                          cudaMemcpyDeviceToHost, st),
                        "D2H U rows");
        if (r == 0) {  // sigma and V are identical on every rank (redundant Jacobi)
          engine::check(cudaMemcpyAsync(b.h_sigma, b.d_sigma, n * sizeof(double), cudaMemcpyDeviceToHost, st),
                        "D2H sigma");
          engine::check(cudaMemcpyAsync(out.factors.v.raw(), b.d_v, (size_t)n * n * elt, cudaMemcpyDeviceToHost, st),
                        "D2H V");
        }
        infos[r] = pl.wait();
      } catch (const std::exception& e) {
        errs[r] = e.what();
      }
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < p; ++r)
    if (!errs[r].empty()) throw std::runtime_error("device " + std::to_string(devs[r]) + ": " + errs[r]);
  const mpsvd_exec_info& info = infos[0];
  std::copy(set.parts[0]->h_sigma, set.parts[0]->h_sigma + n, out.factors.sigma.begin());
  raise_device_status(info, cfg.max_sweeps);
  out.eigensolver = choice;
  out.gram_sync_events = 1;  // the one exchange of the partial Grams
  out.gram_blocks = set.parts[0]->plan->nblocks;
  out.jacobi_sweeps = info.sweeps;
  out.jacobi_rotations = (long)info.rotations;
  // device phases: the slowest rank's
  for (int r = 0; r < p; ++r) {
    out.times.gram = std::max(out.times.gram, infos[r].ms_gram * 1e-3);
    out.times.eigen = std::max(out.times.eigen, infos[r].ms_eigen * 1e-3);
    out.times.compute_u = std::max(out.times.compute_u, infos[r].ms_compute_u * 1e-3);
  }
  out.times.total = std::chrono::duration<double>(Clock::now() - t0).count();
  out.times.overlap = out.times.total - out.times.gram - out.times.eigen - out.times.compute_u;
  if (out.times.overlap < 0.0) {
    out.times.total -= out.times.overlap;
    out.times.overlap = 0.0;
  }
  return out;
}

ThinSvdResult run_thin_svd(const DenseMatrix& a, const JacobiConfig& cfg, bool f64,
                           EigensolverChoice choice = EigensolverChoice::TwoSidedJacobi) {
  const auto t0 = Clock::now();
  const long long m = a.rows(), n = a.cols();
  if (cfg.max_sweeps < 1) throw InvalidArgument("max_sweeps must be >= 1");
  require_device();
  {
    const std::vector<int> devs = shard_devices(m);
    const char* force = getenv("MPSVD_SHARD_FORCE");
    if (devs.size() > 1 || (force && force[0] == '1' && !devs.empty()))
      return run_thin_svd_sharded(a, cfg, f64, choice, devs, t0);
  }
  Bundle& b = bundle_for(m, n, f64);
  engine::Plan& p = *b.plan;
  p.set_jacobi(cfg.tol, cfg.max_sweeps);
  p.set_eigensolver(choice == EigensolverChoice::TwoSidedJacobi ? 0 : choice == EigensolverChoice::GramCholSvd ? 1 : 2);
  cudaStream_t st = p.own_stream;
  const Precision wp = f64 ? Precision::Higher : Precision::Working;
  ThinSvdResult out;
  out.factors.u = DenseMatrix::uninitialized(m, n, wp);  // fully overwritten by the D2H copies
  out.factors.v = DenseMatrix::uninitialized(n, n, wp);
  out.factors.sigma.assign(n, 0.0);
  out.factors.precision = wp;
  // H2D of A and D2H of U in row chunks overlapped with the Gram and U
  // kernels (engine.cu, Plan::execute_host); sigma is downloaded through a
  // page-locked staging slot of the plan
  p.execute_host(a.raw(), b.d_a, out.factors.u.raw(), b.d_u, b.h_sigma, b.d_sigma, out.factors.v.raw(), b.d_v, st);
  const mpsvd_exec_info info = p.wait();
  std::copy(b.h_sigma, b.h_sigma + n, out.factors.sigma.begin());
  raise_device_status(info, cfg.max_sweeps);
  out.eigensolver = choice;
  out.gram_sync_events = 1;  // one global combine of the partial Grams
  out.gram_blocks = p.nblocks;
  out.jacobi_sweeps = info.sweeps;
  out.jacobi_rotations = (long)info.rotations;
  out.times.gram = info.ms_gram * 1e-3;
  out.times.eigen = info.ms_eigen * 1e-3;
  out.times.compute_u = info.ms_compute_u * 1e-3;
  out.times.total = std::chrono::duration<double>(Clock::now() - t0).count();
  out.times.overlap = out.times.total - out.times.gram - out.times.eigen - out.times.compute_u;
  if (out.times.overlap < 0.0) {  // event clocks vs host clock granularity
    out.times.total -= out.times.overlap;
    out.times.overlap = 0.0;
  }
  return out;
}

}  // namespace

ThinSvdResult mp_thin_svd(const DenseMatrix& a, EigensolverChoice choice, const JacobiConfig& cfg, int threads) {
  // validation order of proj/src/thinsvd.cpp:52-56
  if (a.precision() != Precision::Working) throw InvalidArgument("mp_thin_svd expects a Working-precision matrix");
  if (a.rows() < a.cols() || a.cols() < 1) throw InvalidArgument("mp_thin_svd: need m >= n >= 1");
  if (threads < 1) throw InvalidArgument("mp_thin_svd: thread count must be positive");
  return run_thin_svd(a, cfg, false, choice);
}

CholQrFactors mp_cholesky_qr(const DenseMatrix& a) {
  // validation of proj/src/thinsvd.cpp:126-129
  if (a.precision() != Precision::Working) throw InvalidArgument("mp_cholesky_qr expects a Working-precision matrix");
  const long long m = a.rows(), n = a.cols();
  if (m < n || n < 1) throw InvalidArgument("mp_cholesky_qr: need m >= n >= 1");
  require_device();
  Bundle& b = bundle_for(m, n, false);
  engine::Plan& p = *b.plan;
  cudaStream_t st = p.own_stream;
  CholQrFactors out{DenseMatrix::uninitialized(m, n, Precision::Working), DenseMatrix(n, n, Precision::Working)};
  engine::check(cudaMemcpyAsync(b.d_a, a.raw(), (size_t)m * n * 4, cudaMemcpyHostToDevice, st), "H2D A");
  p.cholqr(b.d_a, m, b.d_u, m, st);
  engine::check(cudaMemcpyAsync(out.q.raw(), b.d_u, (size_t)m * n * 4, cudaMemcpyDeviceToHost, st), "D2H Q");
  engine::check(cudaMemcpyAsync(out.r.raw(), p.d_x32, (size_t)n * n * 4, cudaMemcpyDeviceToHost, st), "D2H R");
  const mpsvd_exec_info info = p.wait();
  raise_device_status(info, 0);
  return out;
}

ThinSvdResult mp_thin_svd_f64(const DenseMatrix& a, const JacobiConfig& cfg, int threads) {
  if (a.precision() != Precision::Higher) throw InvalidArgument("mp_thin_svd_f64 expects a Higher-precision matrix");
  if (a.rows() < a.cols() || a.cols() < 1) throw InvalidArgument("mp_thin_svd_f64: need m >= n >= 1");
  if (threads < 1) throw InvalidArgument("mp_thin_svd_f64: thread count must be positive");
  return run_thin_svd(a, cfg, true);
}

namespace {
// Jacobi on an uploaded symmetric M (fp64, or double-double as hi/lo);
// outputs sorted, sign-fixed eigenpairs. Used by twosided_jacobi_eig and the
// stage entry point.
void gpu_jacobi(bool dd, const double* m_hi, const double* m_lo, long long n, double tol, int max_sweeps,
                double* lam_hi, double* lam_lo, double* v_hi, double* v_lo, int* sweeps, long long* rotations) {
  require_device();
  if (n < 1) throw InvalidArgument("twosided_jacobi_eig: empty matrix");
  if (max_sweeps < 1) throw InvalidArgument("max_sweeps must be >= 1");
  engine::Plan p(0, n, dd, nullptr);
  p.set_jacobi(tol, max_sweeps);
  cudaStream_t st = p.own_stream;
  const std::size_t nn = (std::size_t)n * n;
  std::vector<double> inter;
  if (dd) {
    inter.resize(2 * nn);
    for (std::size_t k = 0; k < nn; ++k) {
      inter[2 * k] = m_hi[k];
      inter[2 * k + 1] = m_lo ? m_lo[k] : 0.0;
    }
    engine::check(cudaMemcpyAsync(p.d_m, inter.data(), 2 * nn * 8, cudaMemcpyHostToDevice, st), "H2D M");
  } else {
    engine::check(cudaMemcpyAsync(p.d_m, m_hi, nn * 8, cudaMemcpyHostToDevice, st), "H2D M");
  }
  void* d_vfull = nullptr;
  engine::check(cudaMalloc(&d_vfull, nn * 8 * (dd ? 2 : 1)), "cudaMalloc V");
  p.reset_status(st);
  p.eigen(st);
  engine::check(dev::launch_finish(dd, (int)n, p.jws, p.d_perm, p.d_lam_hi, p.d_lam_lo, p.d_sigma_tmp, nullptr,
                                   nullptr, 1, st, d_vfull),
                "finish");
  p.fetch_status(st);
  std::vector<double> vbuf(nn * (dd ? 2 : 1));
  engine::check(cudaMemcpyAsync(vbuf.data(), d_vfull, vbuf.size() * 8, cudaMemcpyDeviceToHost, st), "D2H V");
  engine::check(cudaMemcpyAsync(lam_hi, p.d_lam_hi, n * 8, cudaMemcpyDeviceToHost, st), "D2H lambda");
  std::vector<double> lo(n);
  engine::check(cudaMemcpyAsync(lo.data(), p.d_lam_lo, n * 8, cudaMemcpyDeviceToHost, st), "D2H lambda lo");
  const mpsvd_exec_info info = p.wait();
  cudaFree(d_vfull);
  raise_device_status(info, max_sweeps);
  if (lam_lo) std::memcpy(lam_lo, lo.data(), n * 8);
  if (dd) {
    for (std::size_t k = 0; k < nn; ++k) {
      v_hi[k] = vbuf[2 * k];
      if (v_lo) v_lo[k] = vbuf[2 * k + 1];
    }
  } else {
    std::memcpy(v_hi, vbuf.data(), nn * 8);
    if (v_lo) std::memset(v_lo, 0, nn * 8);
  }
  if (sweeps) *sweeps = info.sweeps;
  if (rotations) *rotations = info.rotations;
}

void gpu_gram(bool f64, const void* a, long long m, long long n, double* m_hi, double* m_lo) {
  require_device();
  if (m < 1 || n < 1) throw InvalidArgument("gram: need m >= 1, n >= 1");
  engine::Plan p(m, n, f64, nullptr);
  cudaStream_t st = p.own_stream;
  const std::size_t elt = f64 ? 8 : 4;
  void* d_a = nullptr;
  engine::check(cudaMalloc(&d_a, m * n * elt), "cudaMalloc A");
  engine::check(cudaMemcpyAsync(d_a, a, m * n * elt, cudaMemcpyHostToDevice, st), "H2D A");
  p.launches = 0;
  p.gram(d_a, m, st);
  const std::size_t nn = (std::size_t)n * n;
  std::vector<double> buf(nn * (f64 ? 2 : 1));
  engine::check(cudaMemcpyAsync(buf.data(), p.d_m, buf.size() * 8, cudaMemcpyDeviceToHost, st), "D2H M");
  engine::check(cudaStreamSynchronize(st), "sync");
  cudaFree(d_a);
  if (f64) {
    for (std::size_t k = 0; k < nn; ++k) {
      m_hi[k] = buf[2 * k];
      if (m_lo) m_lo[k] = buf[2 * k + 1];
    }
  } else {
    std::memcpy(m_hi, buf.data(), nn * 8);
    if (m_lo) std::memset(m_lo, 0, nn * 8);
  }
}
}  // namespace

EigFactors twosided_jacobi_eig(const DenseMatrix& m, const JacobiConfig& cfg, JacobiStats* stats) {
  const index_t n = m.rows();
  if (m.cols() != n) throw InvalidArgument("twosided_jacobi_eig: not square");
  if (n < 1) throw InvalidArgument("twosided_jacobi_eig: empty matrix");
  if (cfg.max_sweeps < 1) throw InvalidArgument("max_sweeps must be >= 1");
  if (m.precision() != Precision::Higher)
    throw InvalidArgument("twosided_jacobi_eig: the GPU path takes a Higher-precision matrix");
  EigFactors out;
  out.precision = Precision::Higher;
  out.lambda.assign(n, 0.0);
  out.v = DenseMatrix(n, n, Precision::Higher);
  int sw = 0;
  long long rot = 0;
  gpu_jacobi(false, m.dptr(), nullptr, n, cfg.tol, cfg.max_sweeps, out.lambda.data(), nullptr, out.v.dptr(),
             nullptr, &sw, &rot);
  if (stats) {
    stats->sweeps = sw;
    stats->rotations = (long)rot;
    stats->pairs_per_sweep = (long)(n * (n - 1) / 2);
  }
  return out;
}

double orth_error(const DenseMatrix& q) {
  const index_t m = q.rows(), n = q.cols();
  if (m < n) throw InvalidArgument("orth_error: rows < cols");
  std::vector<double> g((std::size_t)n * n);
  gpu_gram(q.precision() == Precision::Higher, q.raw(), m, n, g.data(), nullptr);
  double sum = 0.0;
  for (index_t j = 0; j < n; ++j)
    for (index_t i = 0; i <= j; ++i) {
      const double d = g[(std::size_t)j * n + i] - (i == j ? 1.0 : 0.0);
      sum += (i == j) ? d * d : 2.0 * d * d;
    }
  return std::sqrt(sum);
}

double max_rel_sv_error(const std::vector<double>& computed, const std::vector<double>& reference) {
  if (computed.size() != reference.size()) throw InvalidArgument("singular value arrays differ in length");
  double worst = 0.0;
  for (std::size_t i = 0; i < reference.size(); ++i) {
    if (!(reference[i] > 0.0))
      throw InvalidArgument("reference singular value " + std::to_string(i + 1) + " is not positive");
    worst = std::max(worst, std::abs(computed[i] - reference[i]) / reference[i]);
  }
  return worst;
}

// device-resident backward error (bench validation, the host entry below)
BackwardErrorReport backward_error_device(bool f64, const void* d_a, long long lda, const void* d_u, long long ldu,
                                          const double* d_sigma, const void* d_v, long long ldv, long long m,
                                          long long n, cudaStream_t st) {
  BackwardErrorReport rep;
  if (m == 0 || n == 0) return rep;
  double* partial = nullptr;
  unsigned long long* out = nullptr;
  engine::check(cudaMalloc((void**)&partial, dev::backward_partial_elems(m, (int)n) * sizeof(double)),
                "cudaMalloc backward partials");
  engine::check(cudaMalloc((void**)&out, 2 * sizeof(unsigned long long)), "cudaMalloc backward out");
  unsigned long long h[2] = {0, 0};
  cudaError_t e = dev::launch_backward_error(f64, d_a, lda, d_u, ldu, d_sigma, d_v, ldv, m, (int)n, partial, out, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(partial);
  cudaFree(out);
  engine::check(e, "backward error");
  double worst;
  std::memcpy(&worst, &h[0], sizeof(worst));
  rep.max_rel = worst;
  rep.skipped_rows = (index_t)h[1];
  return rep;
}

BackwardErrorReport rowwise_backward_error(const DenseMatrix& a, const DenseMatrix& u,
                                           const std::vector<double>& sigma, const DenseMatrix& v) {
  const index_t m = a.rows(), n = a.cols();
  if (u.rows() != m || u.cols() != n || (index_t)sigma.size() != n || v.rows() != n || v.cols() != n)
    throw InvalidArgument("factor shapes do not match A");
  if (m == 0 || n == 0) return {};
  require_device();
  // one storage type for the kernel: all Working -> float; otherwise every
  // Working operand is widened (exactly) to binary64 first
  const bool f64 = a.precision() == Precision::Higher || u.precision() == Precision::Higher ||
                   v.precision() == Precision::Higher;
  std::vector<double> wide[3];
  auto host_ptr = [&](const DenseMatrix& x, int slot) -> const void* {
    if (!f64 || x.precision() == Precision::Higher) return x.raw();
    const float* f = x.fptr();
    wide[slot].resize((std::size_t)x.size());
    for (std::size_t k = 0; k < wide[slot].size(); ++k) wide[slot][k] = f[k];
    return wide[slot].data();
  };
  const void* ha = host_ptr(a, 0);
  const void* hu = host_ptr(u, 1);
  const void* hv = host_ptr(v, 2);
  const std::size_t elt = f64 ? 8 : 4;
  cudaStream_t st = nullptr;
  engine::check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  void *da = nullptr, *du = nullptr, *dv = nullptr;
  double* ds = nullptr;
  cudaError_t e = cudaMalloc(&da, (std::size_t)m * n * elt);
  if (e == cudaSuccess) e = cudaMalloc(&du, (std::size_t)m * n * elt);
  if (e == cudaSuccess) e = cudaMalloc(&dv, (std::size_t)n * n * elt);
  if (e == cudaSuccess) e = cudaMalloc((void**)&ds, (std::size_t)n * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpyAsync(da, ha, (std::size_t)m * n * elt, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(du, hu, (std::size_t)m * n * elt, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dv, hv, (std::size_t)n * n * elt, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ds, sigma.data(), (std::size_t)n * 8, cudaMemcpyHostToDevice, st);
  BackwardErrorReport rep;
  std::string err;
  if (e != cudaSuccess) {
    err = cudaGetErrorString(e);
  } else {
    try {
      rep = backward_error_device(f64, da, m, du, m, ds, dv, n, m, n, st);
    } catch (const std::exception& ex) {
      err = ex.what();
    }
  }
  cudaFree(da);
  cudaFree(du);
  cudaFree(dv);
  cudaFree(ds);
  cudaStreamDestroy(st);
  if (!err.empty()) throw std::runtime_error("rowwise_backward_error: " + err);
  return rep;
}

// entry points for the C ABI below
void raise_device_status_public(const mpsvd_exec_info& info, int max_sweeps) {
  raise_device_status(info, max_sweeps);
}
void gpu_gram_public(bool f64, const void* a, long long m, long long n, double* m_hi, double* m_lo) {
  gpu_gram(f64, a, m, n, m_hi, m_lo);
}
// the double-double Gram schedule of a plan (parity tests replay K2z with it)
void gpu_gram_schedule_public(long long m, long long n, int cap, int* nsplit, int* nblocks, int* scb, int* bsb,
                              int* ozaki) {
  require_device();
  engine::Plan p(m, n, true, nullptr);
  *ozaki = p.ozaki ? 1 : 0;
  *nsplit = (int)p.splits.size();
  *nblocks = p.nblocks;
  if ((int)p.splits.size() + 1 > cap || p.nblocks + 1 > cap) throw InvalidArgument("schedule: capacity too small");
  for (size_t i = 0; i < p.scb.size(); ++i) scb[i] = p.scb[i];
  for (size_t i = 0; i < p.block_split_begin.size(); ++i) bsb[i] = p.block_split_begin[i];
}
// the binary32 Gram schedule of a plan: K1z on/off, CTA pairs, chunk bounds
void gpu_gram32_schedule_public(long long m, long long n, int cap, int* ozaki, int* npairs, int* nbounds,
                                int64_t* bounds) {
  require_device();
  engine::Plan p(m, n, false, nullptr);
  *ozaki = p.oz32 ? 1 : 0;
  *npairs = p.oz32_pairs;
  *nbounds = (int)p.oz32_bounds.size();
  if ((int)p.oz32_bounds.size() > cap) throw InvalidArgument("schedule: capacity too small");
  for (size_t i = 0; i < p.oz32_bounds.size(); ++i) bounds[i] = p.oz32_bounds[i];
}
// the spectral phase of the one-sided branches on an uploaded fp64 Gram:
// sorted working-precision sigma and V (binary32), as port_onesided_spectral
void gpu_onesided_public(int choice, const double* m_hi, long long n, double tol, int max_sweeps, double* sigma,
                         float* v, int* sweeps, long long* rotations) {
  require_device();
  if (n < 1) throw InvalidArgument("onesided: empty matrix");
  if (max_sweeps < 1) throw InvalidArgument("max_sweeps must be >= 1");
  if (choice != 1 && choice != 2) throw InvalidArgument("choice must be GRAM_CHOL_SVD or ONESIDED_JACOBI_GRAM");
  engine::Plan p(0, n, false, nullptr);
  p.set_jacobi(tol, max_sweeps);
  p.set_eigensolver(choice);
  cudaStream_t st = p.own_stream;
  const std::size_t nn = (std::size_t)n * n;
  engine::check(cudaMemcpyAsync(p.d_m, m_hi, nn * 8, cudaMemcpyHostToDevice, st), "H2D M");
  p.reset_status(st);
  p.eigen(st);
  p.finish(p.d_sigma_tmp, p.d_vwork_tmp, st);
  p.fetch_status(st);
  engine::check(cudaMemcpyAsync(sigma, p.d_sigma_tmp, n * 8, cudaMemcpyDeviceToHost, st), "D2H sigma");
  engine::check(cudaMemcpyAsync(v, p.d_vwork_tmp, nn * 4, cudaMemcpyDeviceToHost, st), "D2H V");
  const mpsvd_exec_info info = p.wait();
  raise_device_status(info, max_sweeps);
  if (sweeps) *sweeps = info.sweeps;
  if (rotations) *rotations = info.rotations;
}

// The multi-GPU exchange's combine kernel (Plan::exchange) on nranks
// host-supplied partials [rank][n x n] (dd: hi and lo planes), one GPU.
void gpu_rank_combine_public(bool dd, const double* part_hi, const double* part_lo, int nranks, long long n,
                             double* m_hi, double* m_lo) {
  const std::size_t nn = (std::size_t)n * n;
  const std::size_t esz = dd ? 2 : 1;
  std::vector<double> buf(nn * esz * nranks);
  for (std::size_t k = 0; k < nn * nranks; ++k) {
    if (dd) {
      buf[2 * k] = part_hi[k];
      buf[2 * k + 1] = part_lo ? part_lo[k] : 0.0;
    } else {
      buf[k] = part_hi[k];
    }
  }
  cudaStream_t st = nullptr;
  engine::check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  void *d_in = nullptr, *d_out = nullptr;
  cudaError_t e = cudaMalloc(&d_in, buf.size() * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_out, nn * esz * 8);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_in, buf.data(), buf.size() * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = dev::launch_block_tree(d_in, nranks, (int)n, d_out, dd, st);
  std::vector<double> res(nn * esz);
  if (e == cudaSuccess) e = cudaMemcpyAsync(res.data(), d_out, res.size() * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d_in);
  cudaFree(d_out);
  cudaStreamDestroy(st);
  engine::check(e, "rank combine");
  for (std::size_t k = 0; k < nn; ++k) {
    m_hi[k] = dd ? res[2 * k] : res[k];
    if (m_lo) m_lo[k] = dd ? res[2 * k + 1] : 0.0;
  }
}

void gpu_jacobi_public(bool dd, const double* m_hi, const double* m_lo, long long n, double tol, int max_sweeps,
                       double* lam_hi, double* lam_lo, double* v_hi, double* v_lo, int* sweeps,
                       long long* rotations) {
  gpu_jacobi(dd, m_hi, m_lo, n, tol, max_sweeps, lam_hi, lam_lo, v_hi, v_lo, sweeps, rotations);
}

}  // namespace mpsvd

// =============================================================================
// C ABI
//
// The opaque handle layouts, fail(), the guarded() exception-to-status
// ladder (same catch order) and require() below follow the reference's C
// surface, proj/src/capi.cpp:15-81 (its from_result is wrap() here): they are
// the observable error contract of the ABI this library replaces, so they
// are kept as the reference writes them. Everything behind them (plan cache,
// host-buffer pipeline, device metrics, multi-GPU sharding) is this library's.
// =============================================================================
struct mpsvd_matrix {
  mpsvd::DenseMatrix m;
};

struct mpsvd_svd_result {
  mpsvd_matrix u, v;
  std::vector<double> sigma;
  double times[5] = {0, 0, 0, 0, 0};
  int sync_events = 0;
  int64_t gram_blocks = 0;
  int qr_baseline = 0;
  int sweeps = 0;
  int64_t rotations = 0;
};

struct mpsvd_comm {
  mpsvd::engine::Comm* c = nullptr;
};

struct mpsvd_plan {
  std::unique_ptr<mpsvd::engine::Plan> p;
};

namespace {

thread_local std::string t_message;
thread_local int64_t t_index = 0;

mpsvd_status fail(mpsvd_status s, const char* msg, int64_t index = 0) {
  t_message = msg;
  t_index = index;
  return s;
}

template <typename F>
mpsvd_status guarded(F&& body) noexcept {
  using namespace mpsvd;
  try {
    t_message.clear();
    t_index = 0;
    body();
    return MPSVD_OK;
  } catch (const InvalidArgument& e) {
    return fail(MPSVD_ERR_INVALID_ARGUMENT, e.what());
  } catch (const NotPositiveDefiniteError& e) {
    return fail(MPSVD_ERR_NOT_POSITIVE_DEFINITE, e.what(), e.pivot);
  } catch (const NoConvergenceError& e) {
    return fail(MPSVD_ERR_NO_CONVERGENCE, e.what());
  } catch (const ZeroColumnError& e) {
    return fail(MPSVD_ERR_ZERO_COLUMN, e.what(), e.column);
  } catch (const ZeroDivisorError& e) {
    return fail(MPSVD_ERR_ZERO_DIVISOR, e.what(), e.index);
  } catch (const CastOverflowError& e) {
    return fail(MPSVD_ERR_CAST_OVERFLOW, e.what());
  } catch (const TinySingularValueError& e) {
    return fail(MPSVD_ERR_TINY_SINGULAR_VALUE, e.what(), e.index);
  } catch (const InfeasibleError& e) {
    return fail(MPSVD_ERR_INFEASIBLE, e.what());
  } catch (const IoError& e) {
    return fail(MPSVD_ERR_IO, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(MPSVD_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::exception& e) {
    return fail(MPSVD_ERR_INTERNAL, e.what());
  } catch (...) {
    return fail(MPSVD_ERR_INTERNAL, "unknown error");
  }
}

void require(bool ok, const char* msg) {
  if (!ok) throw mpsvd::InvalidArgument(msg);
}

mpsvd_svd_result* wrap(mpsvd::ThinSvdResult&& r) {
  auto* out = new mpsvd_svd_result;
  out->u.m = std::move(r.factors.u);
  out->v.m = std::move(r.factors.v);
  out->sigma = std::move(r.factors.sigma);
  out->times[0] = r.times.gram;
  out->times[1] = r.times.eigen;
  out->times[2] = r.times.compute_u;
  out->times[3] = r.times.overlap;
  out->times[4] = r.times.total;
  out->sync_events = r.gram_sync_events;
  out->gram_blocks = r.gram_blocks;
  out->qr_baseline = r.qr_baseline ? 1 : 0;
  out->sweeps = r.jacobi_sweeps;
  out->rotations = r.jacobi_rotations;
  return out;
}

}  // namespace

extern "C" {

const char* mpsvd_last_error_message(void) { return t_message.c_str(); }
int64_t mpsvd_last_error_index(void) { return t_index; }

mpsvd_status mpsvd_matrix_create(int64_t rows, int64_t cols, mpsvd_precision prec, mpsvd_matrix** out) {
  return guarded([&] {
    require(out != nullptr, "out is null");
    require(rows >= 0 && cols >= 0, "negative dimension");
    require(prec == MPSVD_PRECISION_WORKING || prec == MPSVD_PRECISION_HIGHER, "unknown precision value");
    *out = new mpsvd_matrix{mpsvd::DenseMatrix(
        rows, cols, prec == MPSVD_PRECISION_WORKING ? mpsvd::Precision::Working : mpsvd::Precision::Higher)};
  });
}

void mpsvd_matrix_destroy(mpsvd_matrix* a) { delete a; }
int64_t mpsvd_matrix_rows(const mpsvd_matrix* a) { return a ? a->m.rows() : 0; }
int64_t mpsvd_matrix_cols(const mpsvd_matrix* a) { return a ? a->m.cols() : 0; }
mpsvd_precision mpsvd_matrix_precision(const mpsvd_matrix* a) {
  return (a && a->m.precision() == mpsvd::Precision::Higher) ? MPSVD_PRECISION_HIGHER : MPSVD_PRECISION_WORKING;
}

mpsvd_status mpsvd_matrix_set(mpsvd_matrix* a, int64_t row, int64_t col, double value) {
  return guarded([&] {
    require(a != nullptr, "matrix is null");
    require(row >= 0 && row < a->m.rows() && col >= 0 && col < a->m.cols(), "index out of range");
    a->m.set(row, col, value);
  });
}

mpsvd_status mpsvd_matrix_get(const mpsvd_matrix* a, int64_t row, int64_t col, double* value) {
  return guarded([&] {
    require(a != nullptr && value != nullptr, "null argument");
    require(row >= 0 && row < a->m.rows() && col >= 0 && col < a->m.cols(), "index out of range");
    *value = a->m.get(row, col);
  });
}

int mpsvd_matrix_bitwise_equal(const mpsvd_matrix* a, const mpsvd_matrix* b) {
  if (!a || !b) return 0;
  return a->m.bitwise_equal(b->m) ? 1 : 0;
}

void* mpsvd_matrix_data(mpsvd_matrix* a) { return a ? a->m.raw() : nullptr; }

mpsvd_status mpsvd_orth_error(const mpsvd_matrix* a, double* out) {
  return guarded([&] {
    require(a != nullptr && out != nullptr, "null argument");
    *out = mpsvd::orth_error(a->m);
  });
}

mpsvd_status mpsvd_max_rel_sv_error(const double* computed, const double* reference, int64_t count, double* out) {
  return guarded([&] {
    require(computed != nullptr && reference != nullptr && out != nullptr, "null argument");
    require(count >= 0, "negative count");
    *out = mpsvd::max_rel_sv_error(std::vector<double>(computed, computed + count),
                                   std::vector<double>(reference, reference + count));
  });
}

mpsvd_status mpsvd_rowwise_backward_error(const mpsvd_matrix* a, const mpsvd_matrix* u, const double* sigma,
                                          int64_t count, const mpsvd_matrix* v, double* max_rel,
                                          int64_t* skipped_rows) {
  return guarded([&] {
    require(a != nullptr && u != nullptr && v != nullptr && max_rel != nullptr, "null argument");
    require(count >= 0 && (sigma != nullptr || count == 0), "bad sigma");
    const auto rep = mpsvd::rowwise_backward_error(a->m, u->m, std::vector<double>(sigma, sigma + count), v->m);
    *max_rel = rep.max_rel;
    if (skipped_rows) *skipped_rows = rep.skipped_rows;
  });
}

mpsvd_status mpsvd_backward_error_device(mpsvd_precision prec, const void* d_a, int64_t lda, const void* d_u,
                                         int64_t ldu, const double* d_sigma, const void* d_v, int64_t ldv,
                                         int64_t m, int64_t n, void* stream, double* max_rel, int64_t* skipped_rows) {
  return guarded([&] {
    require(max_rel != nullptr, "null argument");
    require(m >= 0 && n >= 0 && lda >= m && ldu >= m && ldv >= n, "bad shape / leading dimension");
    require(m == 0 || n == 0 || (d_a && d_u && d_sigma && d_v), "null device pointer");
    mpsvd::require_device();
    const auto rep = mpsvd::backward_error_device(prec == MPSVD_PRECISION_HIGHER, d_a, lda, d_u, ldu, d_sigma, d_v,
                                                  ldv, m, n, (cudaStream_t)stream);
    *max_rel = rep.max_rel;
    if (skipped_rows) *skipped_rows = rep.skipped_rows;
  });
}

mpsvd_status mpsvd_thin_svd(const mpsvd_matrix* a, mpsvd_eigensolver eig, int threads, mpsvd_svd_result** out) {
  return guarded([&] {
    require(a != nullptr && out != nullptr, "null argument");
    require(eig == MPSVD_EIG_TWOSIDED_JACOBI || eig == MPSVD_EIG_GRAM_CHOL_SVD || eig == MPSVD_EIG_ONESIDED_JACOBI_GRAM,
            "unknown eigensolver value");
    auto choice = eig == MPSVD_EIG_TWOSIDED_JACOBI ? mpsvd::EigensolverChoice::TwoSidedJacobi
                  : eig == MPSVD_EIG_GRAM_CHOL_SVD ? mpsvd::EigensolverChoice::GramCholSvd
                                                   : mpsvd::EigensolverChoice::OneSidedJacobiOnGram;
    *out = wrap(mpsvd::mp_thin_svd(a->m, choice, {}, threads));
  });
}

mpsvd_status mpsvd_cholesky_qr(const mpsvd_matrix* a, mpsvd_matrix** q_out, mpsvd_matrix** r_out) {
  return guarded([&] {
    require(a != nullptr && q_out != nullptr && r_out != nullptr, "null argument");
    auto f = mpsvd::mp_cholesky_qr(a->m);
    *q_out = new mpsvd_matrix{std::move(f.q)};
    *r_out = new mpsvd_matrix{std::move(f.r)};
  });
}

mpsvd_status mpsvd_plan_cholesky_qr(mpsvd_plan* p, const void* d_a, int64_t lda, void* d_q, int64_t ldq, float* d_r,
                                    void* stream) {
  return guarded([&] {
    require(p != nullptr && p->p, "null plan");
    require(!p->p->dd, "cholesky QR takes a MPSVD_PRECISION_WORKING plan");
    require(lda >= p->p->m && ldq >= p->p->m, "leading dimension too small");
    cudaStream_t st = stream ? (cudaStream_t)stream : p->p->own_stream;
    p->p->cholqr(d_a, lda, d_q, ldq, st);
    if (d_r)
      mpsvd::engine::check(cudaMemcpyAsync(d_r, p->p->d_x32, (size_t)p->p->n * p->p->n * 4, cudaMemcpyDeviceToDevice, st),
                           "R copy");
  });
}

mpsvd_status mpsvd_thin_svd_f64(const mpsvd_matrix* a, int threads, mpsvd_svd_result** out) {
  return guarded([&] {
    require(a != nullptr && out != nullptr, "null argument");
    *out = wrap(mpsvd::mp_thin_svd_f64(a->m, mpsvd::dd_jacobi_config(), threads));
  });
}

void mpsvd_svd_destroy(mpsvd_svd_result* r) { delete r; }
const mpsvd_matrix* mpsvd_svd_u(const mpsvd_svd_result* r) { return r ? &r->u : nullptr; }
const mpsvd_matrix* mpsvd_svd_v(const mpsvd_svd_result* r) { return r ? &r->v : nullptr; }
const double* mpsvd_svd_sigma(const mpsvd_svd_result* r, int64_t* count) {
  if (count) *count = r ? (int64_t)r->sigma.size() : 0;
  return r ? r->sigma.data() : nullptr;
}
void mpsvd_svd_times(const mpsvd_svd_result* r, double times[5]) {
  if (r && times) std::memcpy(times, r->times, sizeof(r->times));
}
int mpsvd_svd_sync_events(const mpsvd_svd_result* r) { return r ? r->sync_events : 0; }
int64_t mpsvd_svd_gram_blocks(const mpsvd_svd_result* r) { return r ? r->gram_blocks : 0; }
int mpsvd_svd_is_qr_baseline(const mpsvd_svd_result* r) { return r ? r->qr_baseline : 0; }
void mpsvd_svd_jacobi_stats(const mpsvd_svd_result* r, int* sweeps, int64_t* rotations) {
  if (sweeps) *sweeps = r ? r->sweeps : 0;
  if (rotations) *rotations = r ? r->rotations : 0;
}

mpsvd_status mpsvd_comm_unique_id(unsigned char id[128]) {
  return guarded([&] {
    require(id != nullptr, "null argument");
    mpsvd::engine::comm_unique_id(id);
  });
}

mpsvd_status mpsvd_comm_init(const unsigned char id[128], int nranks, int rank, mpsvd_comm** out) {
  return guarded([&] {
    require(id != nullptr && out != nullptr, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    auto* c = new mpsvd_comm;
    c->c = mpsvd::engine::comm_init(id, nranks, rank);
    *out = c;
  });
}

void mpsvd_comm_destroy(mpsvd_comm* c) {
  if (!c) return;
  mpsvd::engine::comm_destroy(c->c);
  delete c;
}

mpsvd_status mpsvd_plan_create(int64_t m_local, int64_t n, mpsvd_precision working, mpsvd_comm* comm,
                               mpsvd_plan** out) {
  return guarded([&] {
    require(out != nullptr, "null argument");
    require(n >= 1 && m_local >= 0, "need n >= 1 and m_local >= 0");
    if (!mpsvd::engine::device_available()) throw std::runtime_error("no CUDA device");
    auto* p = new mpsvd_plan;
    p->p = std::make_unique<mpsvd::engine::Plan>(m_local, n, working == MPSVD_PRECISION_HIGHER,
                                                 comm ? comm->c : nullptr);
    *out = p;
  });
}

mpsvd_status mpsvd_plan_execute(mpsvd_plan* p, const void* d_a, int64_t lda, void* d_u, int64_t ldu, void* d_sigma,
                                void* d_v, void* stream) {
  return guarded([&] {
    require(p != nullptr && p->p, "null plan");
    require(lda >= p->p->m && (d_u == nullptr || ldu >= p->p->m), "leading dimension too small");
    p->p->execute(d_a, lda, d_u, ldu, d_sigma, d_v, (cudaStream_t)stream);
  });
}

mpsvd_status mpsvd_plan_wait(mpsvd_plan* p, mpsvd_exec_info* info) {
  mpsvd_exec_info local;
  std::memset(&local, 0, sizeof(local));
  const mpsvd_status s = guarded([&] {
    require(p != nullptr && p->p, "null plan");
    local = p->p->wait();
    mpsvd::raise_device_status_public(local, p->p->max_sweeps);
  });
  if (info) *info = local;
  return s;
}

void mpsvd_plan_destroy(mpsvd_plan* p) { delete p; }

mpsvd_status mpsvd_stage_gram(mpsvd_precision prec, const void* a, int64_t m, int64_t n, double* m_hi, double* m_lo) {
  return guarded([&] {
    require(a != nullptr && m_hi != nullptr, "null argument");
    mpsvd::gpu_gram_public(prec == MPSVD_PRECISION_HIGHER, a, m, n, m_hi, m_lo);
  });
}

mpsvd_status mpsvd_matrix_write_file(const char* path, const mpsvd_matrix* a) {
  return guarded([&] {
    require(path != nullptr && a != nullptr, "null argument");
    mpsvd::write_matrix_file(path, a->m);
  });
}

mpsvd_status mpsvd_matrix_read_file(const char* path, mpsvd_matrix** out) {
  return guarded([&] {
    require(path != nullptr && out != nullptr, "null argument");
    *out = new mpsvd_matrix{mpsvd::read_matrix_file(path)};
  });
}

mpsvd_status mpsvd_stage_gram_schedule(int64_t m, int64_t n, int cap, int* nsplit, int* nblocks, int* scb, int* bsb,
                                       int* ozaki) {
  return guarded([&] {
    require(nsplit && nblocks && scb && bsb && ozaki, "null argument");
    mpsvd::gpu_gram_schedule_public(m, n, cap, nsplit, nblocks, scb, bsb, ozaki);
  });
}

mpsvd_status mpsvd_stage_gram32_schedule(int64_t m, int64_t n, int cap, int* ozaki, int* npairs, int* nbounds,
                                         int64_t* bounds) {
  return guarded([&] {
    require(ozaki && npairs && nbounds && bounds, "null argument");
    mpsvd::gpu_gram32_schedule_public(m, n, cap, ozaki, npairs, nbounds, bounds);
  });
}

mpsvd_status mpsvd_stage_jacobi(int dd, const double* m_hi, const double* m_lo, int64_t n, double tol, int max_sweeps,
                                double* lam_hi, double* lam_lo, double* v_hi, double* v_lo, int* sweeps,
                                int64_t* rotations) {
  return guarded([&] {
    require(m_hi != nullptr && lam_hi != nullptr && v_hi != nullptr, "null argument");
    long long rot = 0;
    mpsvd::gpu_jacobi_public(dd != 0, m_hi, m_lo, n, tol, max_sweeps, lam_hi, lam_lo, v_hi, v_lo, sweeps, &rot);
    if (rotations) *rotations = rot;
  });
}

mpsvd_status mpsvd_stage_onesided(mpsvd_eigensolver eig, const double* m_hi, int64_t n, double tol, int max_sweeps,
                                  double* sigma, float* v, int* sweeps, int64_t* rotations) {
  return guarded([&] {
    require(m_hi != nullptr && sigma != nullptr && v != nullptr, "null argument");
    long long rot = 0;
    mpsvd::gpu_onesided_public((int)eig, m_hi, n, tol, max_sweeps, sigma, v, sweeps, &rot);
    if (rotations) *rotations = rot;
  });
}

mpsvd_status mpsvd_plan_set_eigensolver(mpsvd_plan* p, mpsvd_eigensolver eig) {
  return guarded([&] {
    require(p != nullptr && p->p, "null plan");
    require(eig == MPSVD_EIG_TWOSIDED_JACOBI || eig == MPSVD_EIG_GRAM_CHOL_SVD || eig == MPSVD_EIG_ONESIDED_JACOBI_GRAM,
            "unknown eigensolver value");
    if (eig != MPSVD_EIG_TWOSIDED_JACOBI && p->p->dd)
      throw mpsvd::InvalidArgument("the one-sided branches take a binary32 working matrix");
    p->p->set_eigensolver((int)eig);
  });
}

double mpsvd_fp64_peak_tflops(int device) {
  if (!mpsvd::engine::device_available()) return 0.0;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return 0.0;
  }
  const double t = mpsvd::dev::measure_fp64_peak_tflops(device);
  cudaSetDevice(prev);  // the caller's current device is left as it was
  return t;
}

size_t mpsvd_format_shortest(double value, char* buf, size_t cap) {
  // proj/include/mpsvd.h:168-171: shortest round-trip decimal, truncated to
  // cap - 1 characters plus NUL; returns the full length
  const std::string s = mpsvd::format_shortest(value);
  if (buf && cap > 0) {
    const size_t k = std::min(s.size(), cap - 1);
    std::memcpy(buf, s.data(), k);
    buf[k] = '\0';
  }
  return s.size();
}

mpsvd_status mpsvd_plan_orth_error(mpsvd_plan* p, const void* d_q, int64_t ldq, void* stream, double* out) {
  return guarded([&] {
    require(p != nullptr && p->p && out != nullptr, "null argument");
    require(ldq >= p->p->m && (d_q != nullptr || p->p->m == 0), "bad Q / leading dimension");
    *out = p->p->orth_error(d_q, std::max<int64_t>(1, ldq), (cudaStream_t)stream);
  });
}

mpsvd_status mpsvd_stage_rank_combine(mpsvd_precision prec, const double* part_hi, const double* part_lo, int nranks,
                                      int64_t n, double* m_hi, double* m_lo) {
  return guarded([&] {
    require(part_hi != nullptr && m_hi != nullptr, "null argument");
    require(nranks >= 1 && nranks <= 16 && n >= 1, "need 1 <= nranks <= 16 and n >= 1");
    mpsvd::require_device();
    mpsvd::gpu_rank_combine_public(prec == MPSVD_PRECISION_HIGHER, part_hi, part_lo, nranks, n, m_hi, m_lo);
  });
}

int mpsvd_device_available(void) { return mpsvd::engine::device_available() ? 1 : 0; }

}  // extern "C"
