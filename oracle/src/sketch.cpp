// TEST INFRASTRUCTURE ONLY (see slra_oracle.hpp). Restates the in-scope
// structured operators of /root/reference/proj/src/sketch.cpp, literally:
// composites transform every row and only then keep the requested ones
// (sketch.cpp:520-529, 558-567), which is what the CPU baseline times.
#include <algorithm>
#include <cmath>

#include <complex>

#include "slra_oracle.hpp"

namespace slra_oracle {

OpCount& op_counter() {  // sketch.cpp:11-14
  thread_local OpCount counter;
  return counter;
}

namespace {

void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

// sketch.cpp:43-69
class PermutationOp final : public SketchOperator {
 public:
  explicit PermutationOp(std::vector<Index> sigma) : sigma_(std::move(sigma)) {
    IndexSet check(sigma_, static_cast<Index>(sigma_.size()));
  }
  Index rows() const override { return static_cast<Index>(sigma_.size()); }
  Index cols() const override { return rows(); }
  std::string kind() const override { return "permutation"; }
  Matrix apply(const Matrix& M) const override {
    require(M.rows() == cols(), "permutation apply: dims");
    Matrix out(rows(), M.cols());
    for (Index j = 0; j < M.cols(); ++j)
      for (Index i = 0; i < rows(); ++i) out(i, j) = M(sigma_[static_cast<size_t>(i)], j);
    return out;
  }
  Matrix apply_transpose(const Matrix& M) const override {
    require(M.rows() == rows(), "permutation apply: dims");
    Matrix out(cols(), M.cols());
    for (Index j = 0; j < M.cols(); ++j)
      for (Index i = 0; i < rows(); ++i) out(sigma_[static_cast<size_t>(i)], j) = M(i, j);
    return out;
  }

 private:
  std::vector<Index> sigma_;
};

// sketch.cpp:73-94
class SignDiagonalOp final : public SketchOperator {
 public:
  explicit SignDiagonalOp(Vector d) : d_(std::move(d)) {
    for (double x : d_) require(std::abs(x) > 1e-12, "sign diagonal: entry too close to 0");
  }
  Index rows() const override { return static_cast<Index>(d_.size()); }
  Index cols() const override { return rows(); }
  std::string kind() const override { return "sign_diagonal"; }
  Matrix apply(const Matrix& M) const override {
    require(M.rows() == rows(), "diagonal apply: dims");
    op_counter().muls += static_cast<unsigned long long>(M.size());
    Matrix out(M.rows(), M.cols());
    for (Index j = 0; j < M.cols(); ++j)
      for (Index i = 0; i < M.rows(); ++i) out(i, j) = d_[static_cast<size_t>(i)] * M(i, j);
    return out;
  }
  Matrix apply_transpose(const Matrix& M) const override { return apply(M); }

 private:
  Vector d_;
};

// sketch.cpp:98-107: rows [r0, r0+len) of X, recursion depth `depth`.
void ah_recurse(Matrix& X, Index r0, Index len, int depth) {
  if (depth == 0) return;
  op_counter().adds += static_cast<unsigned long long>(len * X.cols());
  const Index s = len / 2;
  for (Index j = 0; j < X.cols(); ++j) {
    double* x = X.col(j) + r0;
    for (Index i = 0; i < s; ++i) {
      const double a = x[i];
      x[i] = a + x[i + s];      // X.topRows(s) += X.bottomRows(s)
      x[i + s] = a - x[i + s];  // X.bottomRows(s) = a - X.bottomRows(s)
    }
  }
  ah_recurse(X, r0, s, depth - 1);
  ah_recurse(X, r0 + s, s, depth - 1);
}

// sketch.cpp:109-133
class AbridgedHadamardOp final : public SketchOperator {
 public:
  AbridgedHadamardOp(Index n, int d) : n_(n), d_(d) {
    require(d >= 1, "abridged hadamard: depth >= 1");
    require(n % (Index(1) << d) == 0, "abridged hadamard: 2^d must divide n");
  }
  Index rows() const override { return n_; }
  Index cols() const override { return n_; }
  std::string kind() const override { return "abridged_hadamard"; }
  Matrix apply(const Matrix& M) const override {
    require(M.rows() == n_, "AH apply: dims");
    Matrix X = M;
    ah_recurse(X, 0, n_, d_);
    return X;
  }
  Matrix apply_transpose(const Matrix& M) const override { return apply(M); }

 private:
  Index n_;
  int d_;
};

// sketch.cpp:215-282
class SparseCirculantOp final : public SketchOperator {
 public:
  SparseCirculantOp(Index n, double f, std::vector<std::pair<Index, double>> nz)
      : n_(n), f_(f), nz_(std::move(nz)) {
    require(!nz_.empty() && static_cast<Index>(nz_.size()) <= n, "sparse circulant: 1 <= s <= n");
    for (auto& [k, v] : nz_) {
      require(k >= 0 && k < n, "sparse circulant: position out of range");
      require(v != 0.0, "sparse circulant: zero value");
    }
    all_unit_ = std::abs(std::abs(f_) - 1.0) < 1e-15 &&
                std::all_of(nz_.begin(), nz_.end(), [](const auto& p) { return std::abs(p.second) == 1.0; });
  }
  Index rows() const override { return n_; }
  Index cols() const override { return n_; }
  std::string kind() const override { return "sparse_circulant"; }
  void count(const Matrix& M) const {
    const auto s = static_cast<unsigned long long>(nz_.size());
    const auto sz = static_cast<unsigned long long>(M.size());
    if (all_unit_) {
      op_counter().adds += s * sz;
    } else {
      op_counter().muls += s * sz;
      op_counter().adds += (s - 1) * sz;
    }
  }
  Matrix apply(const Matrix& M) const override {
    require(M.rows() == n_, "sparse circulant apply: dims");
    count(M);
    Matrix out(n_, M.cols());
    for (const auto& [k, v] : nz_) {
      const double vf = v * f_;
      for (Index j = 0; j < M.cols(); ++j) {
        double* o = out.col(j);
        const double* x = M.col(j);
        if (k > 0)
          for (Index i = 0; i < n_ - k; ++i) o[k + i] += v * x[i];   // bottomRows(n-k) += v*topRows
        for (Index i = 0; i < k; ++i) o[i] += vf * x[n_ - k + i];  // topRows(k) += (v f) bottomRows(k)
        if (k == 0)
          for (Index i = 0; i < n_; ++i) o[i] += v * x[i];
      }
    }
    return out;
  }
  Matrix apply_transpose(const Matrix& M) const override {
    require(M.rows() == n_, "sparse circulant apply: dims");
    count(M);
    Matrix out(n_, M.cols());
    for (const auto& [k, v] : nz_) {
      const double vf = v * f_;
      for (Index j = 0; j < M.cols(); ++j) {
        double* o = out.col(j);
        const double* x = M.col(j);
        if (k > 0)
          for (Index i = 0; i < n_ - k; ++i) o[i] += v * x[k + i];  // topRows(n-k) += v*bottomRows
        for (Index i = 0; i < k; ++i) o[n_ - k + i] += vf * x[i];  // bottomRows(k) += (v f) topRows(k)
        if (k == 0)
          for (Index i = 0; i < n_; ++i) o[i] += v * x[i];
      }
    }
    return out;
  }

 private:
  Index n_;
  double f_;
  std::vector<std::pair<Index, double>> nz_;
  bool all_unit_ = false;
};

// sketch.cpp:387-413
class GaussianOp final : public SketchOperator {
 public:
  explicit GaussianOp(Matrix G) : G_(std::move(G)) {}
  Index rows() const override { return G_.rows(); }
  Index cols() const override { return G_.cols(); }
  std::string kind() const override { return "gaussian"; }
  Matrix apply(const Matrix& M) const override {
    require(M.rows() == G_.cols(), "gaussian apply: dims");
    return matmul(G_, M);
  }
  Matrix apply_transpose(const Matrix& M) const override {
    require(M.rows() == G_.rows(), "gaussian apply: dims");
    return matmul_tn(G_, M);
  }

 private:
  Matrix G_;
};

// sketch.cpp:417-442
class SubIdentityOp final : public SketchOperator {
 public:
  SubIdentityOp(IndexSet sel, Index total) : sel_(std::move(sel)), total_(total) {
    require(sel_.bound() == total, "sub-identity: index bound mismatch");
  }
  Index rows() const override { return sel_.size(); }
  Index cols() const override { return total_; }
  std::string kind() const override { return "sub_identity"; }
  Matrix apply(const Matrix& M) const override {
    require(M.rows() == total_, "sub-identity apply: dims");
    return select_rows(M, sel_);
  }
  Matrix apply_transpose(const Matrix& M) const override {
    require(M.rows() == sel_.size(), "sub-identity apply: dims");
    Matrix out(total_, M.cols());
    for (Index j = 0; j < M.cols(); ++j)
      for (Index t = 0; t < sel_.size(); ++t) out(sel_[t], j) = M(t, j);
    return out;
  }

 private:
  IndexSet sel_;
  Index total_;
};

// sketch.cpp:502-543
class ProductOp final : public SketchOperator {
 public:
  explicit ProductOp(std::vector<OpPtr> ops) : ops_(std::move(ops)) {
    require(!ops_.empty(), "product: empty");
    for (size_t i = 0; i + 1 < ops_.size(); ++i)
      require(ops_[i]->cols() == ops_[i + 1]->rows(), "product: dimension mismatch");
  }
  Index rows() const override { return ops_.front()->rows(); }
  Index cols() const override { return ops_.back()->cols(); }
  std::string kind() const override { return "product"; }
  Matrix apply(const Matrix& M) const override {
    Matrix out = M;
    for (size_t i = ops_.size(); i-- > 0;) out = ops_[i]->apply(out);
    return out;
  }
  Matrix apply_transpose(const Matrix& M) const override {
    Matrix out = M;
    for (auto& op : ops_) out = op->apply_transpose(out);
    return out;
  }
  bool is_complex() const override {  // sketch.cpp:511-512, 530-540
    for (auto& o : ops_)
      if (o->is_complex()) return true;
    return false;
  }
  CMatrix apply_complex(const CMatrix& M) const override {
    CMatrix out = M;
    for (size_t i = ops_.size(); i-- > 0;) out = ops_[i]->apply_complex(out);
    return out;
  }
  CMatrix apply_transpose_complex(const CMatrix& M) const override {
    CMatrix out = M;
    for (auto& op : ops_) out = op->apply_transpose_complex(out);
    return out;
  }

 private:
  std::vector<OpPtr> ops_;
};

// sketch.cpp:137-211: abridged Fourier, d radix-2 butterfly levels with
// twiddles exp(i 2 pi k / L), outputs interleaved per level.
using cd = std::complex<double>;
using CRows = std::vector<std::vector<cd>>;  // rows x cols, row-major (rows move as units)

void af_recurse(CRows& X, int depth) {
  if (depth == 0) return;
  const Index s = static_cast<Index>(X.size()) / 2, c = static_cast<Index>(X[0].size());
  CRows u(static_cast<size_t>(s), std::vector<cd>(static_cast<size_t>(c)));
  CRows w = u;
  for (Index i = 0; i < s; ++i)
    for (Index j = 0; j < c; ++j) {
      u[i][j] = X[i][j] + X[i + s][j];
      w[i][j] = X[i][j] - X[i + s][j];
    }
  const double theta = 2.0 * M_PI / static_cast<double>(2 * s);
  for (Index i = 0; i < s; ++i) {
    const cd t = std::exp(cd(0, theta * static_cast<double>(i)));
    for (Index j = 0; j < c; ++j) w[i][j] *= t;
  }
  af_recurse(u, depth - 1);
  af_recurse(w, depth - 1);
  for (Index i = 0; i < s; ++i) {
    X[2 * i] = u[i];
    X[2 * i + 1] = w[i];
  }
}

void af_recurse_transpose(CRows& X, int depth) {
  if (depth == 0) return;
  const Index s = static_cast<Index>(X.size()) / 2, c = static_cast<Index>(X[0].size());
  CRows u(static_cast<size_t>(s)), w(static_cast<size_t>(s));
  for (Index i = 0; i < s; ++i) {
    u[i] = X[2 * i];
    w[i] = X[2 * i + 1];
  }
  af_recurse_transpose(u, depth - 1);
  af_recurse_transpose(w, depth - 1);
  const double theta = 2.0 * M_PI / static_cast<double>(2 * s);
  for (Index i = 0; i < s; ++i) {
    const cd t = std::exp(cd(0, theta * static_cast<double>(i)));
    for (Index j = 0; j < c; ++j) w[i][j] *= t;
  }
  for (Index i = 0; i < s; ++i)
    for (Index j = 0; j < c; ++j) {
      X[i][j] = u[i][j] + w[i][j];
      X[i + s][j] = u[i][j] - w[i][j];
    }
}

CRows to_rows(const CMatrix& M) {
  CRows X(static_cast<size_t>(M.rows()), std::vector<cd>(static_cast<size_t>(M.cols())));
  for (Index i = 0; i < M.rows(); ++i)
    for (Index j = 0; j < M.cols(); ++j) X[i][j] = cd(M.re(i, j), M.im(i, j));
  return X;
}
CMatrix from_rows(const CRows& X, Index cols) {
  CMatrix M{Matrix(static_cast<Index>(X.size()), cols), Matrix(static_cast<Index>(X.size()), cols)};
  for (Index i = 0; i < M.rows(); ++i)
    for (Index j = 0; j < cols; ++j) {
      M.re(i, j) = X[i][j].real();
      M.im(i, j) = X[i][j].imag();
    }
  return M;
}

class AbridgedFourierOp final : public SketchOperator {
 public:
  AbridgedFourierOp(Index n, int d) : n_(n), d_(d) {
    require(d >= 1, "abridged fourier: depth >= 1");
    require(n % (Index(1) << d) == 0, "abridged fourier: 2^d must divide n");
  }
  Index rows() const override { return n_; }
  Index cols() const override { return n_; }
  std::string kind() const override { return "abridged_fourier"; }
  bool is_complex() const override { return true; }
  Matrix apply(const Matrix&) const override {
    throw std::logic_error("abridged fourier is complex; use apply_complex");
  }
  Matrix apply_transpose(const Matrix&) const override {
    throw std::logic_error("abridged fourier is complex; use apply_transpose_complex");
  }
  CMatrix apply_complex(const CMatrix& M) const override {
    require(M.rows() == n_, "AF apply: dims");
    if (M.cols() == 0) return M;
    CRows X = to_rows(M);
    af_recurse(X, d_);
    return from_rows(X, M.cols());
  }
  CMatrix apply_transpose_complex(const CMatrix& M) const override {
    require(M.rows() == n_, "AF apply: dims");
    if (M.cols() == 0) return M;
    CRows X = to_rows(M);
    af_recurse_transpose(X, d_);
    return from_rows(X, M.cols());
  }

 private:
  Index n_;
  int d_;
};

// sketch.cpp:545-583
class ColumnSliceOp final : public SketchOperator {
 public:
  ColumnSliceOp(OpPtr inner, IndexSet columns) : inner_(std::move(inner)), cols_(std::move(columns)) {
    require(cols_.bound() == inner_->cols(), "column slice: bound mismatch");
  }
  Index rows() const override { return inner_->rows(); }
  Index cols() const override { return cols_.size(); }
  std::string kind() const override { return "column_slice"; }
  Matrix apply(const Matrix& M) const override {
    require(M.rows() == cols_.size(), "column slice apply: dims");
    Matrix full(inner_->cols(), M.cols());
    for (Index j = 0; j < M.cols(); ++j)
      for (Index t = 0; t < cols_.size(); ++t) full(cols_[t], j) = M(t, j);
    return inner_->apply(full);
  }
  Matrix apply_transpose(const Matrix& M) const override {
    Matrix full = inner_->apply_transpose(M);
    return select_rows(full, cols_);
  }

 private:
  OpPtr inner_;
  IndexSet cols_;
};

}  // namespace

// sketch.cpp:589-675
OpPtr make_permutation(std::vector<Index> sigma) { return std::make_shared<PermutationOp>(std::move(sigma)); }
OpPtr make_sign_diagonal(Vector d) { return std::make_shared<SignDiagonalOp>(std::move(d)); }
OpPtr make_abridged_hadamard(Index n, int d) { return std::make_shared<AbridgedHadamardOp>(n, d); }
OpPtr make_sparse_circulant(Index n, double f, std::vector<std::pair<Index, double>> nz) {
  return std::make_shared<SparseCirculantOp>(n, f, std::move(nz));
}
// sketch.cpp:286-331: x_1 = v_1, x_i = v_i + b_{i-1} x_{i-1} (lower), the
// mirrored backward recurrence when upper; the transpose runs the other way.
class InverseBidiagonalOp final : public SketchOperator {
 public:
  InverseBidiagonalOp(Vector b, bool lower) : b_(std::move(b)), lower_(lower) {}
  Index rows() const override { return static_cast<Index>(b_.size()) + 1; }
  Index cols() const override { return rows(); }
  std::string kind() const override { return "inverse_bidiagonal"; }
  Matrix apply(const Matrix& M) const override { return run(M, lower_); }
  Matrix apply_transpose(const Matrix& M) const override { return run(M, !lower_); }

 private:
  Matrix run(const Matrix& M, bool forward) const {
    require(M.rows() == rows(), "inverse bidiagonal apply: dims");
    Matrix out = M;
    const Index n = rows();
    for (Index j = 0; j < M.cols(); ++j) {
      if (forward) {
        for (Index i = 1; i < n; ++i) out(i, j) += b_[static_cast<size_t>(i - 1)] * out(i - 1, j);
      } else {
        for (Index i = n - 2; i >= 0; --i) out(i, j) += b_[static_cast<size_t>(i)] * out(i + 1, j);
      }
    }
    return out;
  }
  Vector b_;
  bool lower_;
};

// sketch.cpp:335-383: op = P_1 R_1 ... P_q R_q, R = I - 2 w w^T / (w^T w)
class HouseholderChainOp final : public SketchOperator {
 public:
  HouseholderChainOp(std::vector<Vector> w, std::vector<std::vector<Index>> perms)
      : w_(std::move(w)), perms_(std::move(perms)) {
    require(!w_.empty() && w_.size() == perms_.size(), "householder chain: size mismatch");
    n_ = static_cast<Index>(w_[0].size());
    for (auto& v : w_) {
      double s = 0;
      for (double x : v) s += x * x;
      require(static_cast<Index>(v.size()) == n_ && s > 0, "householder chain: bad reflector");
    }
    for (auto& p : perms_) IndexSet(p, n_);
  }
  Index rows() const override { return n_; }
  Index cols() const override { return n_; }
  std::string kind() const override { return "householder_chain"; }
  Matrix apply(const Matrix& M) const override {
    require(M.rows() == n_, "householder chain apply: dims");
    Matrix X = M;
    for (size_t t = w_.size(); t-- > 0;) {
      reflect(w_[t], X);
      Matrix Y(n_, X.cols());
      for (Index j = 0; j < X.cols(); ++j)
        for (Index i = 0; i < n_; ++i) Y(i, j) = X(perms_[t][static_cast<size_t>(i)], j);
      X = std::move(Y);
    }
    return X;
  }
  Matrix apply_transpose(const Matrix& M) const override {
    require(M.rows() == n_, "householder chain apply: dims");
    Matrix X = M;
    for (size_t t = 0; t < w_.size(); ++t) {
      Matrix Y(n_, X.cols());
      for (Index j = 0; j < X.cols(); ++j)
        for (Index i = 0; i < n_; ++i) Y(perms_[t][static_cast<size_t>(i)], j) = X(i, j);
      reflect(w_[t], Y);
      X = std::move(Y);
    }
    return X;
  }

 private:
  // X -= w ((2 / w^T w) (w^T X))
  static void reflect(const Vector& w, Matrix& X) {
    double ww = 0;
    for (double x : w) ww += x * x;
    const double c = 2.0 / ww;
    for (Index j = 0; j < X.cols(); ++j) {
      double s = 0;
      for (Index i = 0; i < X.rows(); ++i) s += w[static_cast<size_t>(i)] * X(i, j);
      const double cs = c * s;
      for (Index i = 0; i < X.rows(); ++i) X(i, j) -= w[static_cast<size_t>(i)] * cs;
    }
  }
  std::vector<Vector> w_;
  std::vector<std::vector<Index>> perms_;
  Index n_ = 0;
};

OpPtr make_inverse_bidiagonal(Vector subdiag, bool lower) {
  return std::make_shared<InverseBidiagonalOp>(std::move(subdiag), lower);
}
OpPtr make_householder_chain(std::vector<Vector> w, std::vector<std::vector<Index>> perms) {
  return std::make_shared<HouseholderChainOp>(std::move(w), std::move(perms));
}
OpPtr gen_inverse_bidiagonal(Index n, Rng& rng) {  // sketch.cpp:652-656
  Vector b(static_cast<size_t>(n - 1));
  for (Index i = 0; i < n - 1; ++i) b[static_cast<size_t>(i)] = rng.sign();
  return make_inverse_bidiagonal(std::move(b), true);
}
OpPtr gen_householder_chain(Index n, Index q, Rng& rng) {  // sketch.cpp:657-665
  std::vector<Vector> w;
  std::vector<std::vector<Index>> perms;
  for (Index t = 0; t < q; ++t) {
    w.push_back(rng.gaussian_vector(n));
    perms.push_back(rng.permutation(n));
  }
  return make_householder_chain(std::move(w), std::move(perms));
}

// sketch.cpp:446-500: signed sum of equally-shaped operators
class SumOp final : public SketchOperator {
 public:
  SumOp(std::vector<OpPtr> ops, std::vector<int> signs) : ops_(std::move(ops)), signs_(std::move(signs)) {
    require(!ops_.empty() && ops_.size() == signs_.size(), "sum: size mismatch");
    for (auto& op : ops_)
      require(op->rows() == ops_[0]->rows() && op->cols() == ops_[0]->cols(), "sum: dimension mismatch");
    for (int s : signs_) require(s == 1 || s == -1, "sum: signs must be +-1");
  }
  Index rows() const override { return ops_[0]->rows(); }
  Index cols() const override { return ops_[0]->cols(); }
  std::string kind() const override { return "sum"; }
  bool is_complex() const override {
    for (auto& o : ops_)
      if (o->is_complex()) return true;
    return false;
  }
  Matrix apply(const Matrix& M) const override { return run([&](const OpPtr& o) { return o->apply(M); }); }
  Matrix apply_transpose(const Matrix& M) const override {
    return run([&](const OpPtr& o) { return o->apply_transpose(M); });
  }
  CMatrix apply_complex(const CMatrix& M) const override {
    CMatrix out;
    for (size_t i = 0; i < ops_.size(); ++i) {
      CMatrix y = ops_[i]->apply_complex(M);
      acc(out.re, y.re, i);
      acc(out.im, y.im, i);
    }
    return out;
  }
  CMatrix apply_transpose_complex(const CMatrix& M) const override {
    CMatrix out;
    for (size_t i = 0; i < ops_.size(); ++i) {
      CMatrix y = ops_[i]->apply_transpose_complex(M);
      acc(out.re, y.re, i);
      acc(out.im, y.im, i);
    }
    return out;
  }

 private:
  // out = s_0 Y_0, then out += s_i Y_i
  void acc(Matrix& out, const Matrix& y, size_t i) const {
    const double s = static_cast<double>(signs_[i]);
    if (i == 0) {
      out = Matrix(y.rows(), y.cols());
      for (Index e = 0; e < y.size(); ++e) out.v[static_cast<size_t>(e)] = s * y.v[static_cast<size_t>(e)];
    } else {
      for (Index e = 0; e < y.size(); ++e) out.v[static_cast<size_t>(e)] += s * y.v[static_cast<size_t>(e)];
    }
  }
  template <class F>
  Matrix run(F&& f) const {
    Matrix out;
    for (size_t i = 0; i < ops_.size(); ++i) acc(out, f(ops_[i]), i);
    return out;
  }
  std::vector<OpPtr> ops_;
  std::vector<int> signs_;
};

OpPtr make_sum(std::vector<OpPtr> ops, std::vector<int> signs) {
  return std::make_shared<SumOp>(std::move(ops), std::move(signs));
}
OpPtr gen_scaled_diagonal(Index n, Rng& rng) {  // sketch.cpp:640-645
  Vector d(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i)
    d[static_cast<size_t>(i)] = static_cast<double>(rng.sign()) * static_cast<double>(1 + rng.uniform_index(4));
  return make_sign_diagonal(std::move(d));
}

// sketch.cpp:695-791: bidiagonal-product pseudo-Gaussian generator and the KS check
Matrix bidiagonal_factor(Index n, const std::vector<int>& signs) {
  require(static_cast<Index>(signs.size()) == n, "bidiagonal_factor: need n signs");
  Matrix B = Matrix::identity(n, n);
  B(0, n - 1) = signs[0];
  for (Index i = 1; i < n; ++i) B(i, i - 1) = signs[static_cast<size_t>(i)];
  return B;
}
namespace {
struct BidiagFactor {
  std::vector<int> signs;
  std::vector<Index> colperm;
};
std::vector<BidiagFactor> draw_factors(Index n, Index T, Rng& rng) {
  std::vector<BidiagFactor> fs;
  for (Index t = 0; t < T; ++t) {
    BidiagFactor f;
    f.signs.resize(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) f.signs[static_cast<size_t>(i)] = rng.sign();
    f.colperm = rng.permutation(n);
    fs.push_back(std::move(f));
  }
  return fs;
}
Vector factor_times(const BidiagFactor& f, const Vector& x) {
  const Index n = static_cast<Index>(x.size());
  Vector p(static_cast<size_t>(n)), y(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) p[static_cast<size_t>(i)] = x[static_cast<size_t>(f.colperm[static_cast<size_t>(i)])];
  y[0] = p[0] + f.signs[0] * p[static_cast<size_t>(n - 1)];
  for (Index i = 1; i < n; ++i)
    y[static_cast<size_t>(i)] = p[static_cast<size_t>(i)] + f.signs[static_cast<size_t>(i)] * p[static_cast<size_t>(i - 1)];
  return y;
}
}  // namespace
Matrix gen_bidiagonal_product(Index n, Index T, Rng& rng, bool standardize) {
  auto fs = draw_factors(n, T, rng);
  Matrix G(n, n);
  for (Index j = 0; j < n; ++j) {
    Vector v(static_cast<size_t>(n), 0.0);
    v[static_cast<size_t>(j)] = 1.0;
    for (Index t = T; t-- > 0;) v = factor_times(fs[static_cast<size_t>(t)], v);
    for (Index i = 0; i < n; ++i) G(i, j) = v[static_cast<size_t>(i)];
  }
  if (standardize && T > 0) {
    for (Index j = 0; j < n; ++j) {
      double mean = 0;
      for (Index i = 0; i < n; ++i) mean += G(i, j);
      mean /= static_cast<double>(n);
      double var = 0;
      for (Index i = 0; i < n; ++i) var += (G(i, j) - mean) * (G(i, j) - mean);
      var /= static_cast<double>(n);
      if (var > 0)
        for (Index i = 0; i < n; ++i) G(i, j) = (G(i, j) - mean) / std::sqrt(var);
    }
  }
  return G;
}
Vector bidiagonal_product_column(Index n, Index T, Index j, Rng& rng) {
  auto fs = draw_factors(n, T, rng);
  Vector v(static_cast<size_t>(n), 0.0);
  v[static_cast<size_t>(j)] = 1.0;
  for (Index t = T; t-- > 0;) v = factor_times(fs[static_cast<size_t>(t)], v);
  return v;
}
std::pair<double, bool> ks_normality(const std::vector<double>& sample) {
  require(sample.size() >= 30, "ks_normality: need at least 30 samples");
  const auto n = sample.size();
  double mean = 0;
  for (double x : sample) mean += x;
  mean /= static_cast<double>(n);
  double var = 0;
  for (double x : sample) var += (x - mean) * (x - mean);
  var /= static_cast<double>(n);
  if (var <= 0) throw std::invalid_argument("ks_normality: degenerate sample");
  std::vector<double> z(sample);
  for (double& x : z) x = (x - mean) / std::sqrt(var);
  std::sort(z.begin(), z.end());
  double d = 0;
  for (size_t i = 0; i < n; ++i) {
    const double cdf = 0.5 * std::erfc(-z[i] / 1.4142135623730951);
    d = std::max(d, std::abs(cdf - static_cast<double>(i + 1) / static_cast<double>(n)));
    d = std::max(d, std::abs(cdf - static_cast<double>(i) / static_cast<double>(n)));
  }
  return {d, d < 1.36 / std::sqrt(static_cast<double>(n))};
}

OpPtr make_gaussian(Matrix G) { return std::make_shared<GaussianOp>(std::move(G)); }
OpPtr make_sub_identity(IndexSet selected, Index total) {
  return std::make_shared<SubIdentityOp>(std::move(selected), total);
}
OpPtr make_product(std::vector<OpPtr> ops) { return std::make_shared<ProductOp>(std::move(ops)); }
OpPtr take_columns(OpPtr op, IndexSet columns) {
  return std::make_shared<ColumnSliceOp>(std::move(op), std::move(columns));
}
OpPtr take_columns(OpPtr op, Index l, ColumnMode mode, Rng& rng) {
  require(l >= 1 && l <= op->cols(), "take_columns: l out of range");
  std::vector<Index> cols;
  if (mode == ColumnMode::Leftmost) {
    for (Index i = 0; i < l; ++i) cols.push_back(i);
  } else {
    cols = rng.distinct_indices(l, op->cols());
  }
  const Index bound = op->cols();
  return take_columns(std::move(op), IndexSet(std::move(cols), bound));
}
OpPtr gen_permutation(Index n, Rng& rng) { return make_permutation(rng.permutation(n)); }
OpPtr gen_sign_diagonal(Index n, Rng& rng) {
  Vector d(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) d[static_cast<size_t>(i)] = rng.sign();
  return make_sign_diagonal(std::move(d));
}
OpPtr gen_sparse_circulant(Index n, Index s, Rng& rng) {
  std::vector<std::pair<Index, double>> nz;
  for (Index k : rng.distinct_indices(s, n)) nz.emplace_back(k, static_cast<double>(rng.sign()));
  const double f = static_cast<double>(rng.sign());
  return make_sparse_circulant(n, f, std::move(nz));
}
OpPtr gen_gaussian(Index rows, Index cols, Rng& rng) { return make_gaussian(rng.gaussian_matrix(rows, cols)); }
OpPtr gen_aph(Index n, int d, Rng& rng) {
  return make_product({gen_permutation(n, rng), make_abridged_hadamard(n, d)});
}
OpPtr gen_asph(Index n, int d, Rng& rng, bool scaled_diag) {  // sketch.cpp:672-675
  OpPtr diag = scaled_diag ? gen_scaled_diagonal(n, rng) : gen_sign_diagonal(n, rng);
  return make_product({gen_permutation(n, rng), std::move(diag), make_abridged_hadamard(n, d)});
}

// sketch.cpp:679-688
Matrix apply(const SketchOperator& op, const Matrix& M, Side side) {
  if (side == Side::Left) return op.apply(M);
  return op.apply_transpose(M.transpose()).transpose();
}
Matrix materialize(const SketchOperator& op, Index cap) {
  require(op.rows() <= cap && op.cols() <= cap, "materialize: cap exceeded");
  return op.apply(Matrix::identity(op.cols(), op.cols()));
}

OpPtr make_abridged_fourier(Index n, int d) { return std::make_shared<AbridgedFourierOp>(n, d); }

CMatrix materialize_complex(const SketchOperator& op, Index cap) {
  require(op.rows() <= cap && op.cols() <= cap, "materialize: cap exceeded");
  return op.apply_complex(CMatrix{Matrix::identity(op.cols(), op.cols()), Matrix(op.cols(), op.cols())});
}

}  // namespace slra_oracle
