// Remaining public entry points around the CUR / LRA path — restatements of
// /root/reference/proj/src/cur.cpp:170-188 (cynical_cur), :257-276
// (lra_to_top_svd), :278-323 (top_svd_to_cur), linalg.cpp:153-161
// (condition_number), lra.cpp:65-86 (deterministic_error_diagnostic).
// TEST INFRASTRUCTURE: the checker for paper_1611_01391_b200/src/cur_extra.cpp.
#include <cmath>

#include "slra_oracle.hpp"

namespace slra_oracle {

namespace {
Matrix rows_sel(const Matrix& X, const IndexSet& I) { return select_rows(X, I); }
}  // namespace

// linalg.cpp:153-161
double condition_number(const Matrix& A, double rank_tol) {
  const Svd f = svd(A);
  if (f.sigma.empty() || f.sigma[0] == 0.0) throw std::invalid_argument("condition_number: zero matrix");
  const double cut = rank_tol * f.sigma[0];
  size_t rho = 0;
  while (rho < f.sigma.size() && f.sigma[rho] > cut) ++rho;
  return f.sigma[0] / f.sigma[rho - 1];
}

// cur.cpp:170-188
CurDecomposition cynical_cur(const EntryOracle& M, Index p, Index q, Index k, Index l, Index r, Rng& rng) {
  const Index m = M.rows(), n = M.cols();
  if (!(r >= 1 && r <= k && k <= p && p <= m && r <= l && l <= q && q <= n))
    throw std::invalid_argument("cynical_cur: need r <= k <= p <= m, r <= l <= q <= n");
  const IndexSet P(rng.distinct_indices(p, m), m);
  const IndexSet Q(rng.distinct_indices(q, n), n);
  const Matrix B = M.block(P, Q);
  const Svd f = svd(B);
  if (f.sigma[0] <= 0 || f.sigma[static_cast<size_t>(r - 1)] <= 1e-10 * f.sigma[0])
    throw GeneratorRankFailure("cynical_cur: sub-block rank below target");
  const IndexSet rl = select_rows_spanning(f.S.left_cols(r), k, 1.1);
  const IndexSet cl = select_rows_spanning(f.T.left_cols(r), l, 1.1);
  std::vector<Index> I, J;
  for (Index t : rl) I.push_back(P[t]);
  for (Index t : cl) J.push_back(Q[t]);
  return primitive_cur(M, IndexSet(std::move(I), m), IndexSet(std::move(J), n), r);
}

// cur.cpp:257-272
Svd lra_to_top_svd(const Matrix& A, const Matrix& W, const Matrix& B, Index r) {
  if (A.cols() != W.rows() || W.cols() != B.rows()) throw std::invalid_argument("lra_to_top_svd: inner dimension mismatch");
  if (r < 1 || r > std::min(W.rows(), W.cols())) throw std::invalid_argument("lra_to_top_svd: bad rank");
  auto [QA, RA] = thin_qr(A);
  auto [QB, RB] = thin_qr(B.transpose());
  const Svd core = svd(matmul(matmul(RA, W), RB.transpose()));
  if (core.sigma[0] <= 0 || core.sigma[static_cast<size_t>(r - 1)] <= 1e-13 * core.sigma[0])
    throw GeneratorRankFailure("lra_to_top_svd: core rank below target");
  Svd out;
  out.S = matmul(QA, core.S.left_cols(r));
  out.sigma.assign(core.sigma.begin(), core.sigma.begin() + r);
  out.T = matmul(QB, core.T.left_cols(r));
  return out;
}

// cur.cpp:278-323
CurDecomposition top_svd_to_cur(const Svd& f, Index k, Index l, double h, CurSelector selector, Rng& rng) {
  const Index m = f.S.rows(), n = f.T.rows(), r = static_cast<Index>(f.sigma.size());
  (void)m;
  (void)n;
  if (k < r || l < r) throw std::invalid_argument("top_svd_to_cur: need k, l >= r");
  IndexSet I, J;
  if (selector == CurSelector::Deterministic) {
    I = select_rows_spanning(f.S, k, h);
    J = select_rows_spanning(f.T, l, h);
  } else {
    auto sample = [&](const Matrix& X, Index count) {
      std::vector<double> p(static_cast<size_t>(X.rows()));
      double tot = 0;
      for (Index i = 0; i < X.rows(); ++i) {
        double q = 0;
        for (Index j = 0; j < X.cols(); ++j) q += X(i, j) * X(i, j);
        tot += (p[static_cast<size_t>(i)] = q);
      }
      std::vector<Index> picked;
      std::vector<char> used(static_cast<size_t>(X.rows()), 0);
      int guard = 0;
      while (static_cast<Index>(picked.size()) < count) {
        if (++guard > 10000) throw SelectionFailure("top_svd_to_cur: sampling failed to find distinct indices");
        double u = rng.uniform() * tot;
        Index i = 0;
        while (i + 1 < X.rows() && u > p[static_cast<size_t>(i)]) u -= p[static_cast<size_t>(i)], ++i;
        if (!used[static_cast<size_t>(i)]) {
          used[static_cast<size_t>(i)] = 1;
          picked.push_back(i);
        }
      }
      return IndexSet(std::move(picked), X.rows());
    };
    I = sample(f.S, k);
    J = sample(f.T, l);
  }
  const Matrix SI = rows_sel(f.S, I), TJ = rows_sel(f.T, J);
  // pinv(TJ^T) * diag(1 / sigma) * pinv(SI), left to right
  Matrix A = pseudo_inverse(TJ.transpose());
  for (Index j = 0; j < A.cols(); ++j) {
    const double inv = 1.0 / f.sigma[static_cast<size_t>(j)];
    for (Index i = 0; i < A.rows(); ++i) A(i, j) *= inv;
  }
  CurDecomposition c;
  c.r = r;
  c.nucleus = matmul(A, pseudo_inverse(SI));
  c.row_set = std::move(I);
  c.col_set = std::move(J);
  return c;
}

// lra.cpp:65-86
std::pair<double, double> deterministic_error_diagnostic(const Matrix& M, const SketchOperator& H, Index r) {
  if (M.rows() > 512 || M.cols() > 512) throw std::invalid_argument("deterministic_error_diagnostic: dense cap 512 exceeded");
  if (H.rows() != M.cols()) throw std::invalid_argument("diagnostic: H rows != n");
  const Index n = M.cols();
  if (r < 1 || r >= n) throw std::invalid_argument("diagnostic: need 1 <= r < n");
  const Svd f = svd(M);
  const Index p = f.T.cols();
  Matrix T1t(r, n), T2t(p - r, n);
  for (Index i = 0; i < n; ++i) {
    for (Index a = 0; a < r; ++a) T1t(a, i) = f.T(i, a);
    for (Index a = r; a < p; ++a) T2t(a - r, i) = f.T(i, a);
  }
  const Matrix C1 = apply(H, T1t, Side::Right), C2 = apply(H, T2t, Side::Right);
  const double head = f.sigma[static_cast<size_t>(r)];
  Matrix D = C2;
  for (Index j = 0; j < D.cols(); ++j)
    for (Index i = 0; i < D.rows(); ++i) D(i, j) = f.sigma[static_cast<size_t>(r + i)] * C2(i, j);
  const double cross = spectral_norm(matmul(D, pseudo_inverse(C1)));
  const double bound = std::sqrt(head * head + cross * cross);
  const LowRankFactors lr = range_finder(M, H, r, RangeVariant::TruncatedRankR);
  const double achieved = spectral_norm(sub(M, matmul(lr.U, lr.V)));
  return {bound, achieved};
}

}  // namespace slra_oracle
