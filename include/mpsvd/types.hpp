// mpsvd-b200 public C++ types — the host-side surface of the reference's
// proj/include/mpsvd/types.hpp:16-197 (Precision, DenseMatrix, DiagMatrix and
// the error hierarchy), kept source-compatible so callers of mp_thin_svd
// compile unchanged against this library.
//
// DenseMatrix is column-major (entry (i,j) at j*rows+i, types.hpp:175-177);
// get() widens exactly, set() rounds to the storage precision (RNE).
// Storage lives in page-locked host memory when the CUDA driver allows it, so
// the host<->device copies of the GPU path run at full PCIe/NVLink-C2C rate;
// the layout and value semantics are identical either way.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mpsvd {

using index_t = std::int64_t;

enum class Precision { Working, Higher };  // binary32 / binary64

constexpr double unit_roundoff(Precision p) { return p == Precision::Working ? 0x1p-24 : 0x1p-53; }
constexpr const char* precision_tag(Precision p) { return p == Precision::Working ? "f32" : "f64"; }

// ---- errors (1-based indices, as in the reference) -------------------------
struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidArgument : Error {
  using Error::Error;
};
struct NotPositiveDefiniteError : Error {
  NotPositiveDefiniteError(index_t p, double v);
  index_t pivot;
  double value;
};
struct NoConvergenceError : Error {
  NoConvergenceError(int s, double w);
  int sweeps;
  double max_offdiag;
};
struct ZeroColumnError : Error {
  explicit ZeroColumnError(index_t c);
  index_t column;
};
struct ZeroDivisorError : Error {
  explicit ZeroDivisorError(index_t i);
  index_t index;
};
struct CastOverflowError : Error {
  CastOverflowError(index_t r, index_t c, double v);
  index_t row, col;
  double value;
};
struct TinySingularValueError : Error {
  TinySingularValueError(index_t i, double v);
  index_t index;
  double value;
};
struct InfeasibleError : Error {
  using Error::Error;
};
struct IoError : Error {
  using Error::Error;
};

// ---- host buffers -------------------------------------------------------------
namespace detail {
// Page-locked when possible (cudaMallocHost), plain heap otherwise. Zeroed.
struct HostBuffer {
  HostBuffer() = default;
  explicit HostBuffer(std::size_t bytes, bool zero = true);
  HostBuffer(const HostBuffer& o);
  HostBuffer& operator=(const HostBuffer& o);
  HostBuffer(HostBuffer&& o) noexcept;
  HostBuffer& operator=(HostBuffer&& o) noexcept;
  ~HostBuffer();
  void* data() const { return ptr_; }
  std::size_t bytes() const { return bytes_; }

 private:
  void release();
  void* ptr_ = nullptr;
  std::size_t bytes_ = 0;
  bool pinned_ = false;
};
}  // namespace detail

class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(index_t rows, index_t cols, Precision prec);
  static DenseMatrix identity(index_t n, Precision prec);
  // additive: storage left uninitialised (for outputs that are overwritten)
  static DenseMatrix uninitialized(index_t rows, index_t cols, Precision prec);

  index_t rows() const { return rows_; }
  index_t cols() const { return cols_; }
  Precision precision() const { return prec_; }
  index_t size() const { return rows_ * cols_; }

  float* fptr() { return prec_ == Precision::Working ? static_cast<float*>(buf_.data()) : nullptr; }
  const float* fptr() const {
    return prec_ == Precision::Working ? static_cast<const float*>(buf_.data()) : nullptr;
  }
  double* dptr() { return prec_ == Precision::Higher ? static_cast<double*>(buf_.data()) : nullptr; }
  const double* dptr() const {
    return prec_ == Precision::Higher ? static_cast<const double*>(buf_.data()) : nullptr;
  }
  void* raw() { return buf_.data(); }
  const void* raw() const { return buf_.data(); }

  double get(index_t i, index_t j) const;
  void set(index_t i, index_t j, double v);
  bool bitwise_equal(const DenseMatrix& other) const;

 private:
  index_t rows_ = 0, cols_ = 0;
  Precision prec_ = Precision::Higher;
  detail::HostBuffer buf_;
};

struct DiagMatrix {
  std::vector<double> entries;
  Precision precision = Precision::Higher;
  DiagMatrix() = default;
  DiagMatrix(std::vector<double> e, Precision p) : entries(std::move(e)), precision(p) {}
  index_t size() const { return static_cast<index_t>(entries.size()); }
};

}  // namespace mpsvd
