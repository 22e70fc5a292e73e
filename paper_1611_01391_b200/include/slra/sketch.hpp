// Structured sketch operators of /root/reference/proj/include/slra/sketch.hpp
// (in-scope kinds: permutation, sign diagonal, abridged Hadamard, sparse
// f-circulant, sub-identity, product, column slice; Gaussian for tests).
//
// B200 design: an operator is an immutable descriptor. Applying it never
// touches the full n x n action: each output row of op*X (or op^T*X) is
// compiled into a short signed combination of input rows ("row
// expression"), evaluated in exactly the reference's order (nz-list order
// for Z_f, the ah_recurse butterfly for AH), so the device computes only the
// l kept outputs (sketch.cpp:558-567 computes all n, then discards) and the
// result is bit-identical.
#pragma once

#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "slra/linalg.hpp"
#include "slra/matrix.hpp"
#include "slra/rng.hpp"

namespace slra {

enum class Side { Left, Right };
enum class ColumnMode { Leftmost, Random };

/// Output row = combine(coef_s * X(src_s, :)); tree 0 = ordered list sum,
/// 1 = radix-2 butterfly over 2^d leaves picking output leaf q.
struct RowExpr {
  int tree = 0;
  std::vector<Index> src;
  std::vector<double> coef;
  int q = 0;
};

/// A compiled plan: `count` outputs of equal width and tree (slra_cuda.h).
struct SketchPlan {
  int tree = 0;
  Index width = 0;
  Index count = 0;
  std::vector<int64_t> src;   // count x width
  std::vector<double> coef;   // count x width
  std::vector<int32_t> q;     // count
};

/// Complex matrix (reference CMatrix = Eigen::MatrixXcd, matrix.hpp:12) as
/// real and imaginary planes — the layout the device kernels use.
struct CMatrix {
  Matrix re, im;
  Index rows() const { return re.rows(); }
  Index cols() const { return re.cols(); }
};

class SketchOperator {
 public:
  virtual ~SketchOperator() = default;
  /// sketch.hpp:36-43: complex operators (abridged Fourier) and the complex
  /// application; a real operator acts on both planes (sketch.cpp:26-37).
  virtual bool is_complex() const { return false; }
  virtual CMatrix apply_complex(const CMatrix& M) const { return {apply(M.re), apply(M.im)}; }
  virtual CMatrix apply_transpose_complex(const CMatrix& M) const {
    return {apply_transpose(M.re), apply_transpose(M.im)};
  }
  virtual Index rows() const = 0;
  virtual Index cols() const = 0;
  virtual std::string kind() const = 0;
  /// Row `i` of (op * X) as a combination of rows of X.
  virtual RowExpr row_of_apply(Index i) const = 0;
  /// Row `i` of (op^T * X) as a combination of rows of X.
  virtual RowExpr row_of_apply_transpose(Index i) const = 0;
  /// op * M and op^T * M on the device (host in, host out).
  Matrix apply(const Matrix& M) const;
  Matrix apply_transpose(const Matrix& M) const;
  /// False for the operators that are not signed row combinations (the
  /// inverse-bidiagonal scan, the Householder chain, and composites holding
  /// one): they cannot compile to a plan and run apply_device instead.
  virtual bool plannable() const { return true; }
  /// Y = op X (transpose: op^T X) on HBM-resident operands; Y preallocated
  /// (rows() or cols() x X.cols()). Default: the compiled plan.
  virtual void apply_device(const DeviceMatrix& X, bool transpose, DeviceMatrix& Y) const;
  /// Compiled plans, cached (operators are immutable): [0] left, [1] right,
  /// [2] left plan of the transpose. Filled by compile_plan / apply_device.
  mutable std::shared_ptr<const SketchPlan> plan_cache[3];
};

using OpPtr = std::shared_ptr<const SketchOperator>;

OpPtr make_permutation(std::vector<Index> sigma);
OpPtr make_sign_diagonal(Vector d);
OpPtr make_abridged_hadamard(Index n, int d);
OpPtr make_sparse_circulant(Index n, double f, std::vector<std::pair<Index, double>> nonzeros);
OpPtr make_sub_identity(IndexSet selected, Index total);
OpPtr make_product(std::vector<OpPtr> ops);
OpPtr take_columns(OpPtr op, IndexSet columns);
OpPtr take_columns(OpPtr op, Index l, ColumnMode mode, Rng& rng);

/// Dense operator G (reference GaussianOp, used by the tests): full-width
/// list plans, not a hot-path operator.
OpPtr make_gaussian(Matrix G);
OpPtr gen_gaussian(Index rows, Index cols, Rng& rng);

/// sketch.cpp:286-383: inverse unit bidiagonal (a scan) and a chain of
/// permuted Householder reflections: not plans, applied on the device.
OpPtr make_inverse_bidiagonal(Vector subdiag, bool lower = true);
OpPtr make_householder_chain(std::vector<Vector> reflectors, std::vector<std::vector<Index>> perms);
OpPtr gen_inverse_bidiagonal(Index n, Rng& rng);
OpPtr gen_householder_chain(Index n, Index q, Rng& rng);
/// sketch.cpp:137-211: complex abridged Fourier (apply_complex only).
OpPtr make_abridged_fourier(Index n, int d);
CMatrix materialize_complex(const SketchOperator& op, Index cap = 4096);

OpPtr gen_permutation(Index n, Rng& rng);
OpPtr gen_sign_diagonal(Index n, Rng& rng);
OpPtr gen_sparse_circulant(Index n, Index s, Rng& rng);
OpPtr gen_aph(Index n, int d, Rng& rng);
OpPtr gen_asph(Index n, int d, Rng& rng, bool scaled_diag = false);
/// Signed sum of equally-shaped operators (sketch.cpp:446-500; device
/// application + accumulation, never a plan) and the +-{1..4} diagonal.
OpPtr make_sum(std::vector<OpPtr> ops, std::vector<int> signs);
OpPtr gen_scaled_diagonal(Index n, Rng& rng);

/// Plans: the columns of M*op (Side::Right, one output per op column) or the
/// rows of op*W (Side::Left, one output per op row).
SketchPlan compile_plan(const SketchOperator& op, Side side);

/// apply(op, M, Side) of sketch.cpp:679-682 on the device.
Matrix apply(const SketchOperator& op, const Matrix& M, Side side);
Matrix materialize(const SketchOperator& op, Index cap = 4096);

}  // namespace slra
