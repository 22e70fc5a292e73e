// Host containers of the B200 `slra` library. Same names and semantics as
// /root/reference/proj/include/slra/matrix.hpp:10-44 with Eigen replaced by a
// plain column-major FP64 matrix (ld = rows, the Eigen default layout), plus
// DeviceMatrix: an HBM-resident matrix the hot path runs on.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <utility>
#include <vector>

namespace slra {

using Index = std::ptrdiff_t;

/// Dense column-major host matrix (Eigen::MatrixXd stand-in).
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols, double fill = 0.0)
      : r_(rows), c_(cols), v_(static_cast<size_t>(rows * cols), fill) {}
  static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
  static Matrix Identity(Index rows, Index cols);
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i, Index j) { return v_[static_cast<size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<size_t>(i + j * r_)]; }
  Matrix transpose() const;

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};
using Vector = std::vector<double>;

/// Ordered set of distinct zero-based indices into a dimension of size
/// `bound` (matrix.hpp:17-36; validation as linalg.cpp:10-17).
class IndexSet {
 public:
  IndexSet() = default;
  IndexSet(std::vector<Index> idx, Index bound);
  static IndexSet iota(Index count, Index bound);
  Index size() const { return static_cast<Index>(idx_.size()); }
  Index bound() const { return bound_; }
  Index operator[](Index t) const { return idx_[static_cast<size_t>(t)]; }
  const std::vector<Index>& indices() const { return idx_; }
  bool contains(Index i) const;
  auto begin() const { return idx_.begin(); }
  auto end() const { return idx_.end(); }

 private:
  std::vector<Index> idx_;
  Index bound_ = 0;
};

/// FP64 matrix in HBM (column-major, explicit ld). Owning unless wrapped
/// with DeviceMatrix::view().
class DeviceMatrix {
 public:
  DeviceMatrix() = default;
  DeviceMatrix(Index rows, Index cols);  // uninitialised device storage
  static DeviceMatrix upload(const Matrix& M);
  static DeviceMatrix view(double* d_ptr, Index rows, Index cols, Index ld);
  DeviceMatrix(DeviceMatrix&& o) noexcept { *this = std::move(o); }
  DeviceMatrix& operator=(DeviceMatrix&& o) noexcept;
  DeviceMatrix(const DeviceMatrix&) = delete;
  DeviceMatrix& operator=(const DeviceMatrix&) = delete;
  ~DeviceMatrix();
  Matrix download() const;
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index ld() const { return ld_; }
  double* data() const { return p_; }

 private:
  Index r_ = 0, c_ = 0, ld_ = 0;
  double* p_ = nullptr;
  bool owns_ = false;
};

Matrix select_rows(const Matrix& A, const IndexSet& I);
Matrix select_cols(const Matrix& A, const IndexSet& J);
Matrix select_block(const Matrix& A, const IndexSet& I, const IndexSet& J);

}  // namespace slra
