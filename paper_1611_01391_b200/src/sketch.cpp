// Sketch operators as descriptors + the row-expression compiler (see
// include/slra/sketch.hpp). Semantics follow /root/reference/proj/src/sketch.cpp:
// PermutationOp :43-69, SignDiagonalOp :73-94, AbridgedHadamardOp/ah_recurse
// :98-133, SparseCirculantOp :215-282, SubIdentityOp :417-442, ProductOp
// :502-543, ColumnSliceOp :545-583, generators :622-675, apply :679-682.
#include "slra/sketch.hpp"

#include <algorithm>
#include <complex>
#include <cmath>

#include "slra/devbuf.hpp"
#include "slra/errors.hpp"

namespace slra {

namespace {

void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

RowExpr leaf(Index src, double coef) {
  RowExpr e;
  e.tree = SLRA_TREE_LIST;
  e.src = {src};
  e.coef = {coef};
  return e;
}

RowExpr zero_row() { return RowExpr{}; }

bool is_exact(const RowExpr& e) { return e.tree == SLRA_TREE_LIST && e.src.size() <= 1; }

// Substitute every leaf row y of `outer` by sub(y). Composition is exact
// (bit-identical to the reference's sequential application) when either all
// substitutions are single signed rows (exact +-1 maps) or `outer` itself
// is a single signed row.
template <typename F>
RowExpr substitute(const RowExpr& outer, F&& sub) {
  if (is_exact(outer)) {
    if (outer.src.empty()) return zero_row();
    RowExpr inner = sub(outer.src[0]);
    for (auto& c : inner.coef) c *= outer.coef[0];
    return inner;
  }
  RowExpr out;
  out.tree = outer.tree;
  out.q = outer.q;
  for (size_t s = 0; s < outer.src.size(); ++s) {
    RowExpr inner = sub(outer.src[s]);
    require(is_exact(inner), "sketch plan: operator chain has two combining factors (not on the device path)");
    if (inner.src.empty()) {
      if (outer.tree == SLRA_TREE_FWHT) {  // keep the butterfly position as an explicit zero
        out.src.push_back(0);
        out.coef.push_back(0.0);
      }
    } else {
      out.src.push_back(inner.src[0]);
      out.coef.push_back(outer.coef[s] * inner.coef[0]);
    }
  }
  return out;
}

class PermutationOp final : public SketchOperator {
 public:
  explicit PermutationOp(std::vector<Index> sigma) : sigma_(std::move(sigma)), inv_(sigma_.size()) {
    IndexSet check(sigma_, static_cast<Index>(sigma_.size()));
    for (size_t i = 0; i < sigma_.size(); ++i) inv_[static_cast<size_t>(sigma_[i])] = static_cast<Index>(i);
  }
  Index rows() const override { return static_cast<Index>(sigma_.size()); }
  Index cols() const override { return rows(); }
  std::string kind() const override { return "permutation"; }
  // (P x)_i = x_{sigma[i]};  (P^T x)_{sigma[i]} = x_i
  RowExpr row_of_apply(Index i) const override { return leaf(sigma_[static_cast<size_t>(i)], 1.0); }
  RowExpr row_of_apply_transpose(Index i) const override { return leaf(inv_[static_cast<size_t>(i)], 1.0); }

 private:
  std::vector<Index> sigma_, inv_;
};

class SignDiagonalOp final : public SketchOperator {
 public:
  explicit SignDiagonalOp(Vector d) : d_(std::move(d)) {
    for (double x : d_) require(std::abs(x) > 1e-12, "sign diagonal: entry too close to 0");
  }
  Index rows() const override { return static_cast<Index>(d_.size()); }
  Index cols() const override { return rows(); }
  std::string kind() const override { return "sign_diagonal"; }
  RowExpr row_of_apply(Index i) const override { return leaf(i, d_[static_cast<size_t>(i)]); }
  RowExpr row_of_apply_transpose(Index i) const override { return row_of_apply(i); }

 private:
  Vector d_;
};

class AbridgedHadamardOp final : public SketchOperator {
 public:
  AbridgedHadamardOp(Index n, int d) : n_(n), d_(d) {
    require(d >= 1, "abridged hadamard: depth >= 1");
    require(n % (Index(1) << d) == 0, "abridged hadamard: 2^d must divide n");
    require(d <= 4, "abridged hadamard: device plans support depth <= 4");
  }
  Index rows() const override { return n_; }
  Index cols() const override { return n_; }
  std::string kind() const override { return "abridged_hadamard"; }
  // ah_recurse: row i couples rows b + j*g (g = n / 2^d, b = i mod g) through
  // the radix-2 butterfly; the output is leaf q = i / g of that butterfly.
  RowExpr row_of_apply(Index i) const override {
    const Index w = Index(1) << d_, g = n_ / w;
    RowExpr e;
    e.tree = SLRA_TREE_FWHT;
    e.q = static_cast<int>(i / g);
    for (Index j = 0; j < w; ++j) {
      e.src.push_back(i % g + j * g);
      e.coef.push_back(1.0);
    }
    return e;
  }
  RowExpr row_of_apply_transpose(Index i) const override { return row_of_apply(i); }  // symmetric

 private:
  Index n_;
  int d_;
};

class SparseCirculantOp final : public SketchOperator {
 public:
  SparseCirculantOp(Index n, double f, std::vector<std::pair<Index, double>> nz) : n_(n), f_(f), nz_(std::move(nz)) {
    require(!nz_.empty() && static_cast<Index>(nz_.size()) <= n, "sparse circulant: 1 <= s <= n");
    for (auto& [k, v] : nz_) {
      require(k >= 0 && k < n, "sparse circulant: position out of range");
      require(v != 0.0, "sparse circulant: zero value");
    }
  }
  Index rows() const override { return n_; }
  Index cols() const override { return n_; }
  std::string kind() const override { return "sparse_circulant"; }
  // (Z_f^k x)_i = x_{i-k} for i >= k, f * x_{n+i-k} otherwise; nz-list order.
  RowExpr row_of_apply(Index i) const override {
    RowExpr e;
    for (auto& [k, v] : nz_) {
      if (i >= k) {
        e.src.push_back(i - k);
        e.coef.push_back(v);
      } else {
        e.src.push_back(n_ + i - k);
        e.coef.push_back(v * f_);
      }
    }
    return e;
  }
  RowExpr row_of_apply_transpose(Index i) const override {
    RowExpr e;
    for (auto& [k, v] : nz_) {
      if (i < n_ - k) {
        e.src.push_back(i + k);
        e.coef.push_back(v);
      } else {
        e.src.push_back(i + k - n_);
        e.coef.push_back(v * f_);
      }
    }
    return e;
  }

 private:
  Index n_;
  double f_;
  std::vector<std::pair<Index, double>> nz_;
};

class SubIdentityOp final : public SketchOperator {
 public:
  SubIdentityOp(IndexSet sel, Index total) : sel_(std::move(sel)), total_(total), pos_(total, -1) {
    require(sel_.bound() == total, "sub-identity: index bound mismatch");
    for (Index t = 0; t < sel_.size(); ++t) pos_[static_cast<size_t>(sel_[t])] = t;
  }
  Index rows() const override { return sel_.size(); }
  Index cols() const override { return total_; }
  std::string kind() const override { return "sub_identity"; }
  RowExpr row_of_apply(Index t) const override { return leaf(sel_[t], 1.0); }
  RowExpr row_of_apply_transpose(Index j) const override {
    const Index t = pos_[static_cast<size_t>(j)];
    return t < 0 ? zero_row() : leaf(t, 1.0);
  }

 private:
  IndexSet sel_;
  Index total_;
  std::vector<Index> pos_;
};

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
  // op0 (op1 (... X)): row i of op0 over rows of op1(...), and so on.
  RowExpr row_of_apply(Index i) const override {
    RowExpr e = ops_[0]->row_of_apply(i);
    for (size_t k = 1; k < ops_.size(); ++k) e = substitute(e, [&](Index y) { return ops_[k]->row_of_apply(y); });
    return e;
  }
  // (op0 ... opL)^T X = opL^T (... op0^T X)
  RowExpr row_of_apply_transpose(Index i) const override {
    RowExpr e = ops_.back()->row_of_apply_transpose(i);
    for (size_t k = ops_.size() - 1; k-- > 0;)
      e = substitute(e, [&](Index y) { return ops_[k]->row_of_apply_transpose(y); });
    return e;
  }
  bool plannable() const override {
    for (auto& o : ops_)
      if (!o->plannable()) return false;
    return true;
  }
  bool is_complex() const override {  // sketch.cpp:511-540
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
    for (auto& o : ops_) out = o->apply_transpose_complex(out);
    return out;
  }
  // a chain holding a non-plan factor: factor by factor on the device, right
  // to left (the transpose left to right), as the reference applies it
  void apply_device(const DeviceMatrix& X, bool transpose, DeviceMatrix& Y) const override {
    if (plannable()) {
      SketchOperator::apply_device(X, transpose, Y);
      return;
    }
    const size_t L = ops_.size();
    DeviceMatrix cur;
    const DeviceMatrix* in = &X;
    for (size_t s = 0; s < L; ++s) {
      const SketchOperator& f = transpose ? *ops_[s] : *ops_[L - 1 - s];
      if (s + 1 == L) {
        f.apply_device(*in, transpose, Y);
        return;
      }
      DeviceMatrix nxt(transpose ? f.cols() : f.rows(), X.cols());
      f.apply_device(*in, transpose, nxt);
      cur = std::move(nxt);
      in = &cur;
    }
  }

 private:
  std::vector<OpPtr> ops_;
};

class ColumnSliceOp final : public SketchOperator {
 public:
  ColumnSliceOp(OpPtr inner, IndexSet columns) : inner_(std::move(inner)), cols_(std::move(columns)),
                                                 pos_(inner_->cols(), -1) {
    require(cols_.bound() == inner_->cols(), "column slice: bound mismatch");
    for (Index t = 0; t < cols_.size(); ++t) pos_[static_cast<size_t>(cols_[t])] = t;
  }
  Index rows() const override { return inner_->rows(); }
  Index cols() const override { return cols_.size(); }
  std::string kind() const override { return "column_slice"; }
  // apply: inner * (rows of M scattered to positions cols)
  RowExpr row_of_apply(Index i) const override {
    return substitute(inner_->row_of_apply(i), [&](Index y) {
      const Index t = pos_[static_cast<size_t>(y)];
      return t < 0 ? zero_row() : leaf(t, 1.0);
    });
  }
  // apply_transpose: select_rows(inner^T M, cols)
  RowExpr row_of_apply_transpose(Index t) const override { return inner_->row_of_apply_transpose(cols_[t]); }
  bool plannable() const override { return inner_->plannable(); }
  void apply_device(const DeviceMatrix& X, bool transpose, DeviceMatrix& Y) const override {
    if (plannable()) {
      SketchOperator::apply_device(X, transpose, Y);
      return;
    }
    const SubIdentityOp sel(cols_, inner_->cols());  // l x n: picks rows cols_
    DeviceMatrix Z(inner_->cols(), X.cols());
    if (!transpose) {  // inner * (X scattered to the rows cols_)
      sel.apply_device(X, true, Z);
      inner_->apply_device(Z, false, Y);
    } else {  // rows cols_ of inner^T X
      inner_->apply_device(X, true, Z);
      sel.apply_device(Z, false, Y);
    }
  }

 private:
  OpPtr inner_;
  IndexSet cols_;
  std::vector<Index> pos_;
};

// sketch.cpp:286-331: the inverse of a unit bidiagonal matrix, applied as a
// recurrence down (lower) or up (upper) every column (slra_bidiag_scan);
// apply_transpose runs the other direction.
class InverseBidiagonalOp final : public SketchOperator {
 public:
  InverseBidiagonalOp(Vector b, bool lower) : b_(std::move(b)), lower_(lower) {}
  Index rows() const override { return static_cast<Index>(b_.size()) + 1; }
  Index cols() const override { return rows(); }
  std::string kind() const override { return "inverse_bidiagonal"; }
  RowExpr row_of_apply(Index) const override { throw std::logic_error("inverse_bidiagonal: not a plan operator"); }
  RowExpr row_of_apply_transpose(Index) const override {
    throw std::logic_error("inverse_bidiagonal: not a plan operator");
  }
  bool plannable() const override { return false; }
  void apply_device(const DeviceMatrix& X, bool transpose, DeviceMatrix& Y) const override {
    require(X.rows() == rows(), "inverse bidiagonal apply: dims");
    if (!db_.get() && !b_.empty()) db_ = DevBuf<double>(b_);
    check(slra_bidiag_scan(device_context(), X.data(), X.ld(), rows(), X.cols(), db_.get(),
                           (lower_ != transpose) ? 1 : 0, Y.data(), Y.ld()),
          "inverse_bidiagonal");
  }

 private:
  Vector b_;
  bool lower_;
  mutable DevBuf<double> db_;
};

// sketch.cpp:335-383: op = P_1 R_1 ... P_q R_q with R = I - 2 w w^T / w^T w.
// Each reflection is two DMMA GEMMs (s = c w^T X with c = 2 / w^T w, then
// X - w s as a rank-1 update with beta = 1), each permutation a row gather.
class HouseholderChainOp final : public SketchOperator {
 public:
  HouseholderChainOp(std::vector<Vector> w, std::vector<std::vector<Index>> perms)
      : w_(std::move(w)), perms_(std::move(perms)) {
    require(!w_.empty() && w_.size() == perms_.size(), "householder chain: size mismatch");
    n_ = static_cast<Index>(w_[0].size());
    for (auto& v : w_) {
      double ss = 0;
      for (double x : v) ss += x * x;
      require(static_cast<Index>(v.size()) == n_ && ss > 0, "householder chain: bad reflector");
      c_.push_back(2.0 / ss);
    }
    for (auto& p : perms_) {
      IndexSet(p, n_);  // validates
      std::vector<int64_t> inv(static_cast<size_t>(n_));
      for (Index i = 0; i < n_; ++i) inv[static_cast<size_t>(p[static_cast<size_t>(i)])] = i;
      inv_.push_back(std::move(inv));
    }
  }
  Index rows() const override { return n_; }
  Index cols() const override { return n_; }
  std::string kind() const override { return "householder_chain"; }
  RowExpr row_of_apply(Index) const override { throw std::logic_error("householder_chain: not a plan operator"); }
  RowExpr row_of_apply_transpose(Index) const override {
    throw std::logic_error("householder_chain: not a plan operator");
  }
  bool plannable() const override { return false; }
  void apply_device(const DeviceMatrix& X, bool transpose, DeviceMatrix& Y) const override {
    require(X.rows() == n_, "householder chain apply: dims");
    slra_ctx cx = device_context();
    const Index c = X.cols();
    DeviceMatrix A(n_, c), B(n_, c);
    DevBuf<double> s(static_cast<size_t>(c));
    // copies are unit rescalings (one coalesced pass)
    check(slra_scale_rows_cols(cx, X.data(), X.ld(), n_, c, nullptr, nullptr, A.data(), A.ld()), "householder_chain");
    const size_t q = w_.size();
    for (size_t k = 0; k < q; ++k) {
      const size_t t = transpose ? k : q - 1 - k;
      DevBuf<double> w(w_[t]);
      if (!transpose) {
        reflect(cx, w.get(), c_[t], A, s.get());
        DevBuf<int64_t> p(std::vector<int64_t>(perms_[t].begin(), perms_[t].end()));  // Y(i) = X(perm[i])
        check(slra_gather_rows(cx, A.data(), A.ld(), n_, c, p.get(), n_, B.data(), B.ld()), "householder_chain");
      } else {
        DevBuf<int64_t> p(inv_[t]);  // Y(perm[i]) = X(i)  <=>  Y(j) = X(inv[j])
        check(slra_gather_rows(cx, A.data(), A.ld(), n_, c, p.get(), n_, B.data(), B.ld()), "householder_chain");
        reflect(cx, w.get(), c_[t], B, s.get());
      }
      std::swap(A, B);
    }
    check(slra_scale_rows_cols(cx, A.data(), A.ld(), n_, c, nullptr, nullptr, Y.data(), Y.ld()), "householder_chain");
  }

 private:
  // X -= w ((2 / w^T w) (w^T X)): s = c (w^T X) (1 x c), then X + (-1) w s
  static void reflect(slra_ctx cx, const double* w, double cf, DeviceMatrix& X, double* s) {
    const Index n = X.rows(), c = X.cols();
    check(slra_gemm(cx, 1, 0, 1, c, n, cf, w, n, X.data(), X.ld(), 0.0, s, 1), "householder_chain");
    check(slra_gemm(cx, 0, 0, n, c, 1, -1.0, w, n, s, 1, 1.0, X.data(), X.ld()), "householder_chain");
  }
  std::vector<Vector> w_;
  std::vector<std::vector<Index>> perms_;
  std::vector<std::vector<int64_t>> inv_;
  std::vector<double> c_;
  Index n_ = 0;
};

// sketch.cpp:137-211: complex abridged Fourier (slra_af_apply). The twiddle
// tables are the reference's exp(i theta k) with theta = 2 pi / (2 s) per
// level, computed here on the host exactly as the reference computes them.
class AbridgedFourierOp final : public SketchOperator {
 public:
  AbridgedFourierOp(Index n, int d) : n_(n), d_(d) {
    require(d >= 1, "abridged fourier: depth >= 1");
    require(n % (Index(1) << d) == 0, "abridged fourier: 2^d must divide n");
    for (int lv = 0; lv < d; ++lv) {
      const Index s = (n >> lv) / 2;
      const double theta = 2.0 * 3.14159265358979323846 / static_cast<double>(2 * s);
      for (Index i = 0; i < s; ++i) {
        const std::complex<double> t = std::exp(std::complex<double>(0, theta * static_cast<double>(i)));
        twr_.push_back(t.real());
        twi_.push_back(t.imag());
      }
    }
  }
  Index rows() const override { return n_; }
  Index cols() const override { return n_; }
  std::string kind() const override { return "abridged_fourier"; }
  bool is_complex() const override { return true; }
  bool plannable() const override { return false; }
  RowExpr row_of_apply(Index) const override { throw std::logic_error("abridged fourier is complex; use apply_complex"); }
  RowExpr row_of_apply_transpose(Index) const override {
    throw std::logic_error("abridged fourier is complex; use apply_transpose_complex");
  }
  void apply_device(const DeviceMatrix&, bool, DeviceMatrix&) const override {
    throw std::logic_error("abridged fourier is complex; use apply_complex");
  }
  CMatrix apply_complex(const CMatrix& M) const override { return run(M, false); }
  CMatrix apply_transpose_complex(const CMatrix& M) const override { return run(M, true); }

 private:
  CMatrix run(const CMatrix& M, bool transpose) const {
    require(M.rows() == n_ && M.im.rows() == n_ && M.im.cols() == M.cols(), "AF apply: dims");
    if (M.cols() == 0) return M;
    if (!dtw_r_.get()) {
      dtw_r_ = DevBuf<double>(twr_);
      dtw_i_ = DevBuf<double>(twi_);
    }
    DeviceMatrix re = DeviceMatrix::upload(M.re), im = DeviceMatrix::upload(M.im);
    DeviceMatrix ore(n_, M.cols()), oim(n_, M.cols());
    check(slra_af_apply(device_context(), re.data(), im.data(), re.ld(), n_, M.cols(), d_, dtw_r_.get(),
                        dtw_i_.get(), transpose ? 1 : 0, ore.data(), oim.data(), ore.ld()),
          "abridged_fourier");
    return CMatrix{ore.download(), oim.download()};
  }
  Index n_;
  int d_;
  std::vector<double> twr_, twi_;
  mutable DevBuf<double> dtw_r_, dtw_i_;
};

// sketch.cpp:446-500: signed sum of equally-shaped operators. Each term is
// applied on the device and accumulated as out = s_0 Y_0, out += s_i Y_i
// (slra_axpby), the reference's order; a sum is never compiled into a plan
// (a concatenated plan would sum the terms in a different order).
class SumOp final : public SketchOperator {
 public:
  SumOp(std::vector<OpPtr> ops, std::vector<int> signs) : ops_(std::move(ops)), signs_(std::move(signs)) {
    require(!ops_.empty() && ops_.size() == signs_.size(), "sum: size mismatch");
    for (auto& op : ops_)
      require(op->rows() == ops_[0]->rows() && op->cols() == ops_[0]->cols(), "sum: dimension mismatch");
    for (int sg : signs_) require(sg == 1 || sg == -1, "sum: signs must be +-1");
  }
  Index rows() const override { return ops_[0]->rows(); }
  Index cols() const override { return ops_[0]->cols(); }
  std::string kind() const override { return "sum"; }
  RowExpr row_of_apply(Index) const override { throw std::logic_error("sum: not a plan operator"); }
  RowExpr row_of_apply_transpose(Index) const override { throw std::logic_error("sum: not a plan operator"); }
  bool plannable() const override { return false; }
  bool is_complex() const override {
    for (auto& o : ops_)
      if (o->is_complex()) return true;
    return false;
  }
  void apply_device(const DeviceMatrix& X, bool transpose, DeviceMatrix& Y) const override {
    slra_ctx cx = device_context();
    DeviceMatrix T(Y.rows(), Y.cols());
    for (size_t i = 0; i < ops_.size(); ++i) {
      ops_[i]->apply_device(X, transpose, T);
      check(slra_axpby(cx, static_cast<double>(signs_[i]), T.data(), T.ld(), i == 0 ? 0.0 : 1.0, Y.data(), Y.ld(),
                       Y.rows(), Y.cols()),
            "sum");
    }
  }
  CMatrix apply_complex(const CMatrix& M) const override { return accumulate(M, false); }
  CMatrix apply_transpose_complex(const CMatrix& M) const override { return accumulate(M, true); }

 private:
  CMatrix accumulate(const CMatrix& M, bool transpose) const {
    slra_ctx cx = device_context();
    DeviceMatrix ore, oim;
    for (size_t i = 0; i < ops_.size(); ++i) {
      const CMatrix y = transpose ? ops_[i]->apply_transpose_complex(M) : ops_[i]->apply_complex(M);
      DeviceMatrix yr = DeviceMatrix::upload(y.re), yi = DeviceMatrix::upload(y.im);
      if (i == 0) {
        ore = DeviceMatrix(y.rows(), y.cols());
        oim = DeviceMatrix(y.rows(), y.cols());
      }
      const double sg = static_cast<double>(signs_[i]), beta = i == 0 ? 0.0 : 1.0;
      check(slra_axpby(cx, sg, yr.data(), yr.ld(), beta, ore.data(), ore.ld(), y.rows(), y.cols()), "sum");
      check(slra_axpby(cx, sg, yi.data(), yi.ld(), beta, oim.data(), oim.ld(), y.rows(), y.cols()), "sum");
    }
    return CMatrix{ore.download(), oim.download()};
  }
  std::vector<OpPtr> ops_;
  std::vector<int> signs_;
};

}  // namespace

// ---------------------------------------------------------------- factories
OpPtr make_sum(std::vector<OpPtr> ops, std::vector<int> signs) {
  return std::make_shared<SumOp>(std::move(ops), std::move(signs));
}
OpPtr gen_scaled_diagonal(Index n, Rng& rng) {  // sketch.cpp:640-645
  Vector d(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i)
    d[static_cast<size_t>(i)] = static_cast<double>(rng.sign()) * static_cast<double>(1 + rng.uniform_index(4));
  return make_sign_diagonal(std::move(d));
}
OpPtr make_abridged_fourier(Index n, int d) { return std::make_shared<AbridgedFourierOp>(n, d); }

CMatrix materialize_complex(const SketchOperator& op, Index cap) {  // sketch.cpp:690-693
  require(op.rows() <= cap && op.cols() <= cap, "materialize: cap exceeded");
  return op.apply_complex(CMatrix{Matrix::Identity(op.cols(), op.cols()), Matrix(op.cols(), op.cols())});
}
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
OpPtr make_permutation(std::vector<Index> sigma) { return std::make_shared<PermutationOp>(std::move(sigma)); }
OpPtr make_sign_diagonal(Vector d) { return std::make_shared<SignDiagonalOp>(std::move(d)); }
OpPtr make_abridged_hadamard(Index n, int d) { return std::make_shared<AbridgedHadamardOp>(n, d); }
OpPtr make_sparse_circulant(Index n, double f, std::vector<std::pair<Index, double>> nz) {
  return std::make_shared<SparseCirculantOp>(n, f, std::move(nz));
}
// Dense operator (sketch.cpp GaussianOp, tests only): every output is the
// full list combination of the rows, coefficients G(i, :) in column order.
class GaussianOp final : public SketchOperator {
 public:
  explicit GaussianOp(Matrix G) : G_(std::move(G)) {}
  Index rows() const override { return G_.rows(); }
  Index cols() const override { return G_.cols(); }
  std::string kind() const override { return "gaussian"; }
  RowExpr row_of_apply(Index i) const override {
    RowExpr e;
    e.tree = SLRA_TREE_LIST;
    for (Index j = 0; j < G_.cols(); ++j) {
      e.src.push_back(j);
      e.coef.push_back(G_(i, j));
    }
    return e;
  }
  RowExpr row_of_apply_transpose(Index j) const override {
    RowExpr e;
    e.tree = SLRA_TREE_LIST;
    for (Index i = 0; i < G_.rows(); ++i) {
      e.src.push_back(i);
      e.coef.push_back(G_(i, j));
    }
    return e;
  }

 private:
  Matrix G_;
};

OpPtr make_gaussian(Matrix G) { return std::make_shared<GaussianOp>(std::move(G)); }
OpPtr gen_gaussian(Index rows, Index cols, Rng& rng) { return make_gaussian(rng.gaussian_matrix(rows, cols)); }

OpPtr make_sub_identity(IndexSet selected, Index total) {
  return std::make_shared<SubIdentityOp>(std::move(selected), total);
}
OpPtr make_product(std::vector<OpPtr> ops) { return std::make_shared<ProductOp>(std::move(ops)); }
OpPtr take_columns(OpPtr op, IndexSet columns) { return std::make_shared<ColumnSliceOp>(std::move(op), std::move(columns)); }
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

// Generators draw in the reference's order (sketch.cpp:634-675).
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
OpPtr gen_aph(Index n, int d, Rng& rng) { return make_product({gen_permutation(n, rng), make_abridged_hadamard(n, d)}); }
OpPtr gen_asph(Index n, int d, Rng& rng, bool scaled_diag) {
  // drawn before the permutation, as sketch.cpp:672-675
  OpPtr diag = scaled_diag ? gen_scaled_diagonal(n, rng) : gen_sign_diagonal(n, rng);
  return make_product({gen_permutation(n, rng), std::move(diag), make_abridged_hadamard(n, d)});
}

// ---------------------------------------------------------------- plans
static SketchPlan compile_plan_uncached(const SketchOperator& op, Side side);

SketchPlan compile_plan(const SketchOperator& op, Side side) {
  auto& slot = op.plan_cache[side == Side::Left ? 0 : 1];
  if (!slot) slot = std::make_shared<const SketchPlan>(compile_plan_uncached(op, side));
  return *slot;
}

static SketchPlan compile_plan_uncached(const SketchOperator& op, Side side) {
  const Index count = side == Side::Left ? op.rows() : op.cols();
  std::vector<RowExpr> rows;
  rows.reserve(static_cast<size_t>(count));
  int tree = -1;
  Index width = 1;
  for (Index t = 0; t < count; ++t) {
    RowExpr e = side == Side::Left ? op.row_of_apply(t) : op.row_of_apply_transpose(t);
    if (!e.src.empty() || e.tree == SLRA_TREE_FWHT) {
      if (tree < 0) tree = e.tree;
      require(tree == e.tree, "sketch plan: mixed combination trees");
    }
    width = std::max<Index>(width, static_cast<Index>(e.src.size()));
    rows.push_back(std::move(e));
  }
  SketchPlan p;
  p.tree = tree < 0 ? SLRA_TREE_LIST : tree;
  p.width = width;
  p.count = count;
  p.src.assign(static_cast<size_t>(count * width), 0);
  p.coef.assign(static_cast<size_t>(count * width), 0.0);
  p.q.assign(static_cast<size_t>(count), 0);
  for (Index t = 0; t < count; ++t) {
    const RowExpr& e = rows[static_cast<size_t>(t)];
    if (p.tree == SLRA_TREE_FWHT) require(static_cast<Index>(e.src.size()) == width, "sketch plan: ragged butterfly");
    for (size_t s = 0; s < e.src.size(); ++s) {
      p.src[static_cast<size_t>(t * width) + s] = e.src[s];
      p.coef[static_cast<size_t>(t * width) + s] = e.coef[s];
    }
    p.q[static_cast<size_t>(t)] = e.q;
  }
  return p;
}

namespace {

void run_plan_device(const SketchPlan& p, const DeviceMatrix& X, bool rows_mode, DeviceMatrix& out) {
  slra_ctx ctx = device_context();
  DevBuf<int64_t> src(p.src);
  DevBuf<double> coef(p.coef);
  DevBuf<int32_t> q(p.q);
  if (rows_mode)
    check(slra_sketch_rows(ctx, X.data(), X.ld(), X.rows(), X.cols(), src.get(), coef.get(), q.get(), p.width,
                           p.tree, p.count, out.data(), out.ld()),
          "slra_sketch_rows");
  else
    check(slra_sketch_cols(ctx, X.data(), X.ld(), X.rows(), X.cols(), src.get(), coef.get(), q.get(), p.width,
                           p.tree, p.count, out.data(), out.ld()),
          "slra_sketch_cols");
}

// the transpose of an operator as an operator (rows of op^T M: a left plan)
struct TransposeView final : SketchOperator {
  const SketchOperator& o;
  explicit TransposeView(const SketchOperator& x) : o(x) {}
  Index rows() const override { return o.cols(); }
  Index cols() const override { return o.rows(); }
  std::string kind() const override { return "transpose"; }
  RowExpr row_of_apply(Index i) const override { return o.row_of_apply_transpose(i); }
  RowExpr row_of_apply_transpose(Index i) const override { return o.row_of_apply(i); }
};

Matrix host_transpose(const Matrix& M) {  // data movement only
  Matrix T(M.cols(), M.rows());
  for (Index j = 0; j < M.cols(); ++j)
    for (Index i = 0; i < M.rows(); ++i) T(j, i) = M(i, j);
  return T;
}

}  // namespace

void SketchOperator::apply_device(const DeviceMatrix& X, bool transpose, DeviceMatrix& Y) const {
  if (transpose) {
    if (!plan_cache[2]) {
      TransposeView t(*this);
      plan_cache[2] = std::make_shared<const SketchPlan>(compile_plan(t, Side::Left));
    }
    run_plan_device(*plan_cache[2], X, true, Y);
  } else {
    run_plan_device(compile_plan(*this, Side::Left), X, true, Y);
  }
}

Matrix SketchOperator::apply(const Matrix& M) const {
  require(M.rows() == cols(), "sketch apply: dims");
  DeviceMatrix dM = DeviceMatrix::upload(M), out(rows(), M.cols());
  apply_device(dM, false, out);
  return out.download();
}

Matrix SketchOperator::apply_transpose(const Matrix& M) const {
  require(M.rows() == rows(), "sketch apply: dims");
  DeviceMatrix dM = DeviceMatrix::upload(M), out(cols(), M.cols());
  apply_device(dM, true, out);
  return out.download();
}

Matrix apply(const SketchOperator& op, const Matrix& M, Side side) {
  if (side == Side::Left) return op.apply(M);
  // M * op = (op^T M^T)^T: column t of M*op combines columns of M.
  require(M.cols() == op.rows(), "sketch apply: dims");
  if (!op.plannable()) return host_transpose(op.apply_transpose(host_transpose(M)));
  DeviceMatrix dM = DeviceMatrix::upload(M), out(M.rows(), op.cols());
  run_plan_device(compile_plan(op, Side::Right), dM, false, out);
  return out.download();
}

Matrix materialize(const SketchOperator& op, Index cap) {
  require(op.rows() <= cap && op.cols() <= cap, "materialize: cap exceeded");
  return op.apply(Matrix::Identity(op.cols(), op.cols()));
}

}  // namespace slra
