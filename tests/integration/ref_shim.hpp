// Minimal stand-ins for the reference's public types (proj/include/slra/
// matrix.hpp, oracle.hpp, cur.hpp) — just the members the cross_approx
// dispatch of INTEGRATION.md §3 touches — so that the reference-side glue
// (b200.hpp + the SLRA_B200 definition) compiles and runs here without Eigen.
// In the reference these are Eigen::MatrixXd (column-major, ld == rows()),
// IndexSet, EntryOracle and CurDecomposition / CaTrace themselves.
#pragma once

#include <cstddef>
#include <optional>
#include <stdexcept>
#include <vector>

namespace slra {

using Index = std::ptrdiff_t;

struct Matrix {  // Eigen::MatrixXd: column-major, data() contiguous, ld == rows()
  Index r = 0, c = 0;
  std::vector<double> v;
  Matrix() = default;
  Matrix(Index rows, Index cols) : r(rows), c(cols), v(static_cast<size_t>(rows * cols)) {}
  Index rows() const { return r; }
  Index cols() const { return c; }
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  double operator()(Index i, Index j) const { return v[static_cast<size_t>(i + j * r)]; }
};

class IndexSet {  // matrix.hpp:17-36
 public:
  IndexSet() = default;
  IndexSet(std::vector<Index> idx, Index bound) : idx_(std::move(idx)), bound_(bound) {
    for (Index i : idx_)
      if (i < 0 || i >= bound_) throw std::invalid_argument("IndexSet: index out of range");
  }
  Index size() const { return static_cast<Index>(idx_.size()); }
  const std::vector<Index>& indices() const { return idx_; }

 private:
  std::vector<Index> idx_;
  Index bound_ = 0;
};

class EntryOracle {  // oracle.hpp:11-22
 public:
  virtual ~EntryOracle() = default;
  virtual Index rows() const = 0;
  virtual Index cols() const = 0;
  virtual Matrix dense() const = 0;
};
class DenseOracle final : public EntryOracle {
 public:
  explicit DenseOracle(const Matrix& M) : M_(&M) {}
  Index rows() const override { return M_->rows(); }
  Index cols() const override { return M_->cols(); }
  Matrix dense() const override { return *M_; }

 private:
  const Matrix* M_;
};

struct CurDecomposition {  // cur.hpp:16-26
  IndexSet row_set, col_set;
  Matrix nucleus;  // l x k
  Index r = 0;
};
struct CaStep {  // cur.hpp:57-66
  bool horizontal = false;
  std::vector<Index> rows, cols;
  double volume_proxy = 0;
  std::optional<double> error_estimate;
};
struct CaTrace {
  std::vector<CaStep> steps;
};

// the reference's typed failures (errors.hpp:11-33)
struct RangeFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct SketchRankFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct SelectionFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct GeneratorRankFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct PremultRankFailure : std::runtime_error { using std::runtime_error::runtime_error; };

}  // namespace slra
