// slra_oracle — CPU restatement of the reference `slra` hot path.
//
// TEST INFRASTRUCTURE ONLY. This library is the parity checker for the
// B200 path in paper_1611_01391_b200/. Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it; the
// product never links, imports or calls anything under oracle/.
//
// It restates, single-threaded and without Eigen (absent from this image,
// see DESIGN.md "Oracle"), the functions of /root/reference/proj listed in
// SURVEY.md §8(a). Each definition cites the reference file:line it follows.
// Eigen-internal semantics (HouseholderQR, ColPivHouseholderQR, maxCoeff
// traversal order, BDCSVD sign convention) are restated from the published
// Eigen 3.3/3.4 algorithms; BDCSVD itself is replaced by one-sided Jacobi
// (identical singular triplets up to rounding; the reference's own sign
// convention `linalg.cpp:87-96` removes the sign ambiguity).
//
// Parity pin: the reference cannot be compiled here (no Eigen, no vendored
// doctest/CLI11/json: SURVEY.md §8c), and no reference test stores an
// output value of these decompositions. The oracle is pinned against every
// known-answer test the reference holds for the path (tests/test_oracle_*.py
// cite each one) plus the C++ standard's mt19937_64 10000th-draw value and
// LAPACK (scipy) cross-checks. Bitwise equality with the Eigen binary is
// "parity unpinned".
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace slra_oracle {

using Index = std::ptrdiff_t;  // Eigen::Index (matrix.hpp:14)

// ---------------------------------------------------------------- containers
// Column-major dense matrix, ld = rows (Eigen default, matrix.hpp:10).
struct Matrix {
  Index r = 0, c = 0;
  std::vector<double> v;
  Matrix() = default;
  Matrix(Index rows, Index cols, double fill = 0.0)
      : r(rows), c(cols), v(static_cast<size_t>(rows * cols), fill) {}
  Index rows() const { return r; }
  Index cols() const { return c; }
  Index size() const { return r * c; }
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  double& operator()(Index i, Index j) { return v[static_cast<size_t>(i + j * r)]; }
  double operator()(Index i, Index j) const { return v[static_cast<size_t>(i + j * r)]; }
  double* col(Index j) { return v.data() + j * r; }
  const double* col(Index j) const { return v.data() + j * r; }
  static Matrix identity(Index rows, Index cols);
  Matrix transpose() const;
  Matrix left_cols(Index n) const;
  Matrix top_rows(Index n) const;
};
using Vector = std::vector<double>;

// matrix.hpp:17-36, linalg.cpp:10-29
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

// errors.hpp:11-33
struct RangeFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct SketchRankFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct PremultRankFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct SelectionFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct GeneratorRankFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct EmptySample : std::runtime_error { using std::runtime_error::runtime_error; };

// ---------------------------------------------------------------- Rng
// rng.hpp:14-49, rng.cpp:8-66
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : eng_(seed) {}
  std::uint64_t next_u64() { return eng_(); }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double gaussian();
  Index uniform_index(Index n);
  int sign() { return (next_u64() & 1u) ? 1 : -1; }
  std::vector<Index> permutation(Index n);
  std::vector<Index> distinct_indices(Index k, Index n);
  Matrix gaussian_matrix(Index rows, Index cols);
  Vector gaussian_vector(Index n);
  static std::uint64_t derive_seed(std::uint64_t master, std::uint64_t stream);
  Rng child(std::uint64_t stream) { return Rng(derive_seed(next_u64(), stream)); }

 private:
  std::mt19937_64 eng_;
};

// ---------------------------------------------------------------- linalg
// linalg.hpp:11-53
struct Svd {
  Matrix S;
  Vector sigma;
  Matrix T;
};
struct LowRankFactors {
  Matrix U, V;
  Index target_rank = 0;
};
enum class RankMode { Absolute, Relative };
enum class NormKind { Spectral, Frobenius, Chebyshev };

Matrix matmul(const Matrix& A, const Matrix& B);            // linalg.cpp:63-66
Matrix matmul_tn(const Matrix& A, const Matrix& B);         // A^T B
Matrix sub(const Matrix& A, const Matrix& B);               // A - B
Matrix select_rows(const Matrix& A, const IndexSet& I);     // linalg.cpp:35-39
Matrix select_cols(const Matrix& A, const IndexSet& J);     // linalg.cpp:41-45
Matrix select_block(const Matrix& A, const IndexSet& I, const IndexSet& J);  // :47-52
std::pair<Matrix, Matrix> thin_qr(const Matrix& A);         // linalg.cpp:67-79
Svd svd(const Matrix& A);                                   // linalg.cpp:81-98
LowRankFactors truncate_rank(const Matrix& A, Index rho);   // linalg.cpp:100-109
Matrix pseudo_inverse(const Matrix& A, double rank_tol = 1e-10);  // :111-121
Index numerical_rank(const Matrix& A, double tol, RankMode mode = RankMode::Absolute);  // :123-132
double spectral_norm(const Matrix& A);                      // :134-137
double frobenius_norm(const Matrix& A);                     // :139
double chebyshev_norm(const Matrix& A);                     // :141-143
double matrix_norm(const Matrix& A, NormKind kind);         // :145-151
double determinant_abs(const Matrix& A);                    // Eigen PartialPivLU det (cur.cpp:192-197)

// Eigen::ColPivHouseholderQR restated (used at cur.cpp:95,103 and lsr.cpp:52).
struct ColPivQR {
  Matrix qr;                  // R above the diagonal, essential Householder parts below
  Vector hcoeffs;             // tau_k
  std::vector<Index> perm;    // colsPermutation().indices()
  Index nonzero_pivots = 0;
  double maxpivot = 0;
  double threshold = -1;      // < 0: Eigen default eps * diagSize
  explicit ColPivQR(const Matrix& A);
  Index rank() const;
  Matrix solve(const Matrix& B) const;  // least-squares / exact solve, Eigen _solve_impl
};
// Eigen CompleteOrthogonalDecomposition(G) + setThreshold + pseudoInverse
// (cur.cpp:146-152); *rank = cod.rank() at `threshold`.
Matrix cod_pseudo_inverse(const Matrix& G, double threshold, Index* rank);

// ---------------------------------------------------------------- oracles
// oracle.hpp:11-54, testgen.cpp:11-37
class EntryOracle {
 public:
  virtual ~EntryOracle() = default;
  virtual Index rows() const = 0;
  virtual Index cols() const = 0;
  virtual double entry(Index i, Index j) const = 0;
  Matrix rows_of(const IndexSet& I) const;
  Matrix cols_of(const IndexSet& J) const;
  Matrix block(const IndexSet& I, const IndexSet& J) const;
  Matrix dense() const;
};
class DenseOracle final : public EntryOracle {
 public:
  explicit DenseOracle(const Matrix& M) : M_(&M) {}
  Index rows() const override { return M_->rows(); }
  Index cols() const override { return M_->cols(); }
  double entry(Index i, Index j) const override {
    ++accesses_;
    return (*M_)(i, j);
  }
  unsigned long long accesses() const { return accesses_; }
  void reset_accesses() { accesses_ = 0; }

 private:
  const Matrix* M_;
  mutable unsigned long long accesses_ = 0;
};
class FunctionOracle final : public EntryOracle {
 public:
  FunctionOracle(Index rows, Index cols, std::function<double(Index, Index)> f)
      : rows_(rows), cols_(cols), f_(std::move(f)) {}
  Index rows() const override { return rows_; }
  Index cols() const override { return cols_; }
  double entry(Index i, Index j) const override { return f_(i, j); }

 private:
  Index rows_, cols_;
  std::function<double(Index, Index)> f_;
};

// ---------------------------------------------------------------- sketch
// sketch.hpp:15-89; in-scope kinds only.
enum class Side { Left, Right };
enum class ColumnMode { Leftmost, Random };
struct OpCount {
  unsigned long long adds = 0, muls = 0;
  unsigned long long total() const { return adds + muls; }
};
OpCount& op_counter();
inline void reset_op_counter() { op_counter() = OpCount{}; }

// Complex matrices as real and imaginary planes (Eigen::MatrixXcd, matrix.hpp:12);
// element arithmetic goes through std::complex<double>.
struct CMatrix {
  Matrix re, im;
  Index rows() const { return re.rows(); }
  Index cols() const { return re.cols(); }
};

class SketchOperator {
 public:
  virtual ~SketchOperator() = default;
  virtual Index rows() const = 0;
  virtual Index cols() const = 0;
  virtual std::string kind() const = 0;
  virtual Matrix apply(const Matrix& M) const = 0;
  virtual Matrix apply_transpose(const Matrix& M) const = 0;
  // sketch.hpp:36-43, sketch.cpp:26-37: a real operator acts on both parts
  virtual bool is_complex() const { return false; }
  virtual CMatrix apply_complex(const CMatrix& M) const { return {apply(M.re), apply(M.im)}; }
  virtual CMatrix apply_transpose_complex(const CMatrix& M) const {
    return {apply_transpose(M.re), apply_transpose(M.im)};
  }
};
using OpPtr = std::shared_ptr<const SketchOperator>;

OpPtr make_permutation(std::vector<Index> sigma);
OpPtr make_sign_diagonal(Vector d);
OpPtr make_abridged_hadamard(Index n, int d);
OpPtr make_sparse_circulant(Index n, double f, std::vector<std::pair<Index, double>> nz);
OpPtr make_gaussian(Matrix G);
OpPtr make_inverse_bidiagonal(Vector subdiag, bool lower = true);                      // sketch.cpp:286-331
OpPtr make_householder_chain(std::vector<Vector> w, std::vector<std::vector<Index>> perms);  // :335-383
OpPtr gen_inverse_bidiagonal(Index n, Rng& rng);
OpPtr gen_householder_chain(Index n, Index q, Rng& rng);
OpPtr make_sub_identity(IndexSet selected, Index total);
OpPtr make_product(std::vector<OpPtr> ops);
OpPtr make_sum(std::vector<OpPtr> ops, std::vector<int> signs);                 // sketch.cpp:446-500
OpPtr gen_scaled_diagonal(Index n, Rng& rng);                                   // :640-645
Matrix bidiagonal_factor(Index n, const std::vector<int>& signs);               // :697-703
Matrix gen_bidiagonal_product(Index n, Index T, Rng& rng, bool standardize = true);  // :740-758
Vector bidiagonal_product_column(Index n, Index T, Index j, Rng& rng);           // :760-766
std::pair<double, bool> ks_normality(const std::vector<double>& sample);         // :768-791
OpPtr take_columns(OpPtr op, IndexSet columns);
OpPtr take_columns(OpPtr op, Index l, ColumnMode mode, Rng& rng);
OpPtr gen_permutation(Index n, Rng& rng);
OpPtr gen_sign_diagonal(Index n, Rng& rng);
OpPtr gen_sparse_circulant(Index n, Index s, Rng& rng);
OpPtr gen_gaussian(Index rows, Index cols, Rng& rng);
OpPtr gen_aph(Index n, int d, Rng& rng);
OpPtr gen_asph(Index n, int d, Rng& rng, bool scaled_diag = false);
Matrix apply(const SketchOperator& op, const Matrix& M, Side side);
Matrix materialize(const SketchOperator& op, Index cap = 4096);
OpPtr make_abridged_fourier(Index n, int d);                                   // sketch.cpp:137-211
CMatrix materialize_complex(const SketchOperator& op, Index cap = 4096);      // sketch.cpp:690-693

// ---------------------------------------------------------------- cur
// cur.hpp:16-73
struct CurDecomposition {
  IndexSet row_set, col_set;
  Matrix nucleus;  // l x k
  Index r = 0;
};
struct CaStep {
  bool horizontal = false;
  std::vector<Index> rows, cols;
  double volume_proxy = 0;
  std::optional<double> error_estimate;
};
struct CaTrace {
  std::vector<CaStep> steps;
};
Matrix cur_reconstruct(const Matrix& M, const CurDecomposition& c);
double cur_evaluate(const Matrix& M, const CurDecomposition& c, NormKind norm);
double t_factor(Index q, Index s, double h);
enum class CurSelector { Deterministic, Sampled };
CurDecomposition cynical_cur(const EntryOracle& M, Index p, Index q, Index k, Index l, Index r, Rng& rng);
CurDecomposition top_svd_to_cur(const Svd& f, Index k, Index l, double h, CurSelector selector, Rng& rng);
double condition_number(const Matrix& A, double rank_tol = 1e-10);
IndexSet maxvol_rows(const Matrix& A, double h = 1.1, Index max_swaps = 0);
IndexSet select_rows_spanning(const Matrix& A, Index count, double h = 1.1);
CurDecomposition primitive_cur(const EntryOracle& M, IndexSet I, IndexSet J, Index r, bool qr_nucleus = false);
CurDecomposition primitive_cur(const Matrix& M, IndexSet I, IndexSet J, Index r, bool qr_nucleus = false);
std::pair<CurDecomposition, CaTrace> cross_approx(const EntryOracle& M, Index r, Index k, Index l,
                                                  IndexSet init_rows, int loops, double h,
                                                  std::optional<double> stop_tol, Rng& rng);

// ---------------------------------------------------------------- lra
enum class RangeVariant { BasisQr, TruncatedRankR };
LowRankFactors range_finder(const Matrix& M, const SketchOperator& H, Index r,
                            RangeVariant variant = RangeVariant::BasisQr);
LowRankFactors two_stage_truncate(const LowRankFactors& f, Index r);
LowRankFactors lra_premult(const Matrix& M, const SketchOperator& F, const SketchOperator& H, Index r,
                           RangeVariant variant = RangeVariant::BasisQr);
struct LraErrorEstimate {
  double estimate_frobenius = 0;
  Index sample_rows = 0, sample_cols = 0;
  double ci_lo = 0, ci_hi = 0;
  bool has_interval = false;
};
LraErrorEstimate posterior_error_estimate(const EntryOracle& M, const LowRankFactors& f, Index q,
                                          Index s, Rng& rng);

// ---------------------------------------------------------------- lsr
struct LsrProblem {
  Matrix A;
  Vector b;
};
struct LsrReport {
  Vector x_hat;
  double sketched_residual = 0;
  std::optional<double> true_residual, ratio;
  Index k = 0;
  bool validated = true;
  int attempts = 1;
};
Vector solve_exact(const LsrProblem& p);
double residual_norm(const LsrProblem& p, const Vector& x);
double residual_ratio(const LsrProblem& p, const Vector& x_hat);
LsrReport sketch_solve(const LsrProblem& p, const SketchOperator& F, bool with_true_residual = false);
LsrReport solve_with_retries(const LsrProblem& p, OpPtr base_F, const std::vector<OpPtr>& q_family,
                             int max_retries, double accept_tol, Rng& rng);  // lsr.cpp:69-113

// ---------------------------------------------------------------- leverage
// leverage.hpp:11-70, cur.hpp (lra_to_top_svd)
struct LeverageScores {
  Vector p;
  double beta = 1.0;
  Index r = 0;
};
struct SampleRescale {
  std::vector<Index> indices;
  Vector d;
};
enum class SampleMode { Exactly, Expected };
LeverageScores svd_leverage_scores(const Matrix& T_r, double beta = 1.0);
SampleRescale sample_exactly(const LeverageScores& scores, Index l, Rng& rng);
SampleRescale sample_expected(const LeverageScores& scores, Index l, Rng& rng);
SampleRescale collapse_duplicates(const SampleRescale& s);
CurDecomposition cur_via_leverage(const EntryOracle& M, Index r, Index k, Index l, double beta, double beta_bar,
                                  SampleMode mode, const std::optional<LeverageScores>& scores, Rng& rng,
                                  bool plain_nucleus = false);
Svd lra_to_top_svd(const LowRankFactors& f, Index r);
Svd lra_to_top_svd(const Matrix& A, const Matrix& W, const Matrix& B, Index r);
std::pair<double, double> deterministic_error_diagnostic(const Matrix& M, const SketchOperator& H, Index r);
CurDecomposition refine_lra(const EntryOracle& M, const LowRankFactors& crude, Index r, Index k, Index l, Rng& rng);
LeverageScores uniform_scores(Index n);
double gaussian_score_gap(const Matrix& G);
double sample_bound_quadratic(Index r, double eps, double beta);
double sample_bound_loglinear(Index r, double eps, double beta, double cbar);
double epsilon_for_sample(Index r, Index l, double delta);

// ---------------------------------------------------------------- hss
// hss.hpp:11-52
struct HssBlock {
  Index row0 = 0, col0 = 0, rows = 0, cols = 0;
  Matrix F, H;
  bool rank_overflow = false;
};
struct HssLeaf {
  Index row0 = 0, col0 = 0;
  Matrix D;
};
struct HssMatrix {
  Index n = 0;
  int depth = 0;
  Index leaf = 0, r = 0;
  std::vector<HssLeaf> diag;
  std::vector<HssBlock> off;
  bool any_overflow = false;
};
enum class HssStrategy { Svd, CurCa };
HssMatrix build_hss(const EntryOracle& M, int L, Index r, double tol, HssStrategy strategy, Rng& rng);
Vector hss_matvec(const HssMatrix& H, const Vector& x);
Matrix hss_reconstruct(const HssMatrix& H);
double hss_error(const HssMatrix& H, const Matrix& M, NormKind norm);

// ---------------------------------------------------------------- testgen
Matrix random_orthonormal(Index rows, Index cols, Rng& rng);                  // testgen.cpp:41-43
Matrix gen_svd_profile(Index n, Index r, Rng& rng);                           // :100-108
Matrix gen_factor_gaussian(Index m, Index n, Index r, double noise, Rng& rng);  // :110-115
LsrProblem gen_lsr_gaussian(Index m, Index n, double noise, Rng& rng);       // :159-193 (Gaussian)

}  // namespace slra_oracle
