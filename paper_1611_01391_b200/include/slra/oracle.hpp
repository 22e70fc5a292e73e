// Entry-access views (/root/reference/proj/include/slra/oracle.hpp:11-54).
// The device path needs the matrix in HBM: DenseOracle uploads its host
// matrix once (cached) and counts the entries the algorithm reads, exactly
// as the reference's access counter would; DeviceOracle wraps HBM-resident
// data with no copy.
#pragma once

#include <memory>

#include "slra/matrix.hpp"

namespace slra {

class EntryOracle {
 public:
  virtual ~EntryOracle() = default;
  virtual Index rows() const = 0;
  virtual Index cols() const = 0;
  /// HBM view the kernels read (uploading on first use when needed).
  virtual const DeviceMatrix& device() const = 0;
  /// Record `n` algorithmic entry reads (the reference's DenseOracle counter).
  virtual void count(unsigned long long n) const { (void)n; }
};

class DenseOracle final : public EntryOracle {
 public:
  explicit DenseOracle(const Matrix& M) : M_(&M) {}
  Index rows() const override { return M_->rows(); }
  Index cols() const override { return M_->cols(); }
  const DeviceMatrix& device() const override;
  void count(unsigned long long n) const override { accesses_ += n; }
  unsigned long long accesses() const { return accesses_; }
  void reset_accesses() { accesses_ = 0; }

 private:
  const Matrix* M_;
  mutable std::unique_ptr<DeviceMatrix> dev_;
  mutable unsigned long long accesses_ = 0;
};

class DeviceOracle final : public EntryOracle {
 public:
  DeviceOracle(double* d_ptr, Index rows, Index cols, Index ld)
      : view_(DeviceMatrix::view(d_ptr, rows, cols, ld)) {}
  Index rows() const override { return view_.rows(); }
  Index cols() const override { return view_.cols(); }
  const DeviceMatrix& device() const override { return view_; }

 private:
  DeviceMatrix view_;
};

}  // namespace slra
