// The remaining public entry points around the CUR / LRA path
// (/root/reference/proj/src/cur.cpp:170-188, 257-323; linalg.cpp:100-109,
// 153-161; lra.cpp:65-127; cur_evaluate's spectral / Chebyshev norms),
// composed from the device primitives: SVDs, pivoted selections, gathers,
// pseudo-inverses, GEMMs and norms run on the device; the host draws from the
// caller's Rng and evaluates the reference's scalar formulas.
#include <cmath>

#include "slra/cur.hpp"
#include "slra/devbuf.hpp"
#include "slra/errors.hpp"
#include "slra/lra.hpp"

namespace slra {

namespace {
std::vector<int64_t> to64(const IndexSet& s) { return std::vector<int64_t>(s.begin(), s.end()); }

Matrix left_cols(const Matrix& A, Index r) {
  Matrix out(A.rows(), r);
  for (Index j = 0; j < r; ++j)
    for (Index i = 0; i < A.rows(); ++i) out(i, j) = A(i, j);
  return out;
}

Matrix transpose(const Matrix& A) {  // data movement
  Matrix T(A.cols(), A.rows());
  for (Index j = 0; j < A.cols(); ++j)
    for (Index i = 0; i < A.rows(); ++i) T(j, i) = A(i, j);
  return T;
}
}  // namespace

LowRankFactors truncate_rank(const Matrix& A, Index rho) {  // linalg.cpp:100-109
  if (rho < 1 || rho > std::min(A.rows(), A.cols())) throw std::invalid_argument("truncate_rank: rho out of range");
  const Index p = std::min(A.rows(), A.cols());
  slra_ctx cx = device_context();
  DeviceMatrix dA = DeviceMatrix::upload(A), S(A.rows(), p), T(A.cols(), p), U(A.rows(), rho), V(rho, A.cols());
  DevBuf<double> sig(static_cast<size_t>(p));
  check(slra_svd(cx, dA.data(), dA.ld(), A.rows(), A.cols(), S.data(), S.ld(), sig.get(), T.data(), T.ld()),
        "truncate_rank");
  check(slra_scale_rows_cols(cx, S.data(), S.ld(), A.rows(), rho, nullptr, sig.get(), U.data(), U.ld()),
        "truncate_rank");
  check(slra_transpose(cx, T.data(), T.ld(), A.cols(), rho, V.data(), V.ld()), "truncate_rank");
  LowRankFactors f;
  f.U = U.download();
  f.V = V.download();
  f.target_rank = rho;
  return f;
}

double condition_number(const Matrix& A, double rank_tol) {  // linalg.cpp:153-161
  const Svd f = svd(A);
  if (f.sigma.empty() || f.sigma[0] == 0.0) throw std::invalid_argument("condition_number: zero matrix");
  const double cut = rank_tol * f.sigma[0];
  size_t rho = 0;
  while (rho < f.sigma.size() && f.sigma[rho] > cut) ++rho;
  return f.sigma[0] / f.sigma[rho - 1];
}

// cur.cpp:170-188: a random p x q sub-block, its top-r singular factors,
// maxvol selections inside them, then primitive_cur on the full matrix
CurDecomposition cynical_cur(const EntryOracle& M, Index p, Index q, Index k, Index l, Index r, Rng& rng) {
  const Index m = M.rows(), n = M.cols();
  if (!(r >= 1 && r <= k && k <= p && p <= m && r <= l && l <= q && q <= n))
    throw std::invalid_argument("cynical_cur: need r <= k <= p <= m, r <= l <= q <= n");
  const IndexSet P(rng.distinct_indices(p, m), m);
  const IndexSet Q(rng.distinct_indices(q, n), n);
  const DeviceMatrix& dA = M.device();
  DevBuf<int64_t> dP(to64(P)), dQ(to64(Q));
  DeviceMatrix B(p, q);
  check(slra_gather_block(device_context(), dA.data(), dA.ld(), m, n, dP.get(), p, dQ.get(), q, B.data(), B.ld()),
        "cynical_cur");
  M.count(static_cast<unsigned long long>(p * q));
  const Svd f = svd(B.download());
  if (f.sigma[0] <= 0 || f.sigma[static_cast<size_t>(r - 1)] <= 1e-10 * f.sigma[0])
    throw GeneratorRankFailure("cynical_cur: sub-block rank below target");
  const IndexSet rl = select_rows_spanning(left_cols(f.S, r), k, 1.1);
  const IndexSet cl = select_rows_spanning(left_cols(f.T, r), l, 1.1);
  std::vector<Index> I, J;
  for (Index t : rl) I.push_back(P[t]);
  for (Index t : cl) J.push_back(Q[t]);
  return primitive_cur(M, IndexSet(std::move(I), m), IndexSet(std::move(J), n), r);
}

// cur.cpp:257-272 (general W)
Svd lra_to_top_svd(const Matrix& A, const Matrix& W, const Matrix& B, Index r) {
  if (A.cols() != W.rows() || W.cols() != B.rows()) throw std::invalid_argument("lra_to_top_svd: inner dimension mismatch");
  if (r < 1 || r > std::min(W.rows(), W.cols())) throw std::invalid_argument("lra_to_top_svd: bad rank");
  auto [QA, RA] = thin_qr(A);
  auto [QB, RB] = thin_qr(transpose(B));
  const Svd core = svd(matmul(matmul(RA, W), transpose(RB)));
  if (core.sigma[0] <= 0 || core.sigma[static_cast<size_t>(r - 1)] <= 1e-13 * core.sigma[0])
    throw GeneratorRankFailure("lra_to_top_svd: core rank below target");
  Svd out;
  out.S = matmul(QA, left_cols(core.S, r));
  out.sigma.assign(core.sigma.begin(), core.sigma.begin() + r);
  out.T = matmul(QB, left_cols(core.T, r));
  return out;
}

// cur.cpp:278-323
CurDecomposition top_svd_to_cur(const Svd& f, Index k, Index l, double h, CurSelector selector, Rng& rng) {
  const Index r = static_cast<Index>(f.sigma.size());
  if (k < r || l < r) throw std::invalid_argument("top_svd_to_cur: need k, l >= r");
  IndexSet I, J;
  if (selector == CurSelector::Deterministic) {
    I = select_rows_spanning(f.S, k, h);
    J = select_rows_spanning(f.T, l, h);
  } else {
    // norm-square sampling: row weights on the device, the draws on the host
    auto sample = [&](const Matrix& X, Index count) {
      DeviceMatrix dX = DeviceMatrix::upload(X);
      DevBuf<double> dp(static_cast<size_t>(X.rows()));
      check(slra_row_sqnorms(device_context(), dX.data(), dX.ld(), X.rows(), X.cols(), 1.0, dp.get()),
            "top_svd_to_cur");
      const std::vector<double> p = dp.download();
      double tot = 0;
      for (double v : p) tot += v;
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
  // nucleus = pinv(T_J^T) diag(1 / sigma) pinv(S_I), left to right
  Matrix A = pseudo_inverse(transpose(select_rows(f.T, J)));  // l x r
  std::vector<double> inv(static_cast<size_t>(r));
  for (Index j = 0; j < r; ++j) inv[static_cast<size_t>(j)] = 1.0 / f.sigma[static_cast<size_t>(j)];
  DeviceMatrix dA = DeviceMatrix::upload(A);
  DevBuf<double> dinv(inv);
  check(slra_scale_rows_cols(device_context(), dA.data(), dA.ld(), A.rows(), r, nullptr, dinv.get(), dA.data(),
                             dA.ld()),
        "top_svd_to_cur");
  CurDecomposition c;
  c.r = r;
  c.nucleus = matmul(dA.download(), pseudo_inverse(select_rows(f.S, I)));
  c.row_set = std::move(I);
  c.col_set = std::move(J);
  return c;
}

// lra.cpp:65-86 (dense cap 512)
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
  DeviceMatrix dC2 = DeviceMatrix::upload(C2);
  DevBuf<double> tail(std::vector<double>(f.sigma.begin() + r, f.sigma.end()));
  check(slra_scale_rows_cols(device_context(), dC2.data(), dC2.ld(), C2.rows(), C2.cols(), tail.get(), nullptr,
                             dC2.data(), dC2.ld()),
        "deterministic_error_diagnostic");
  const double cross = spectral_norm(matmul(dC2.download(), pseudo_inverse(C1)));
  const double bound = std::sqrt(head * head + cross * cross);
  const LowRankFactors lr = range_finder(M, H, r, RangeVariant::TruncatedRankR);
  DeviceMatrix dM = DeviceMatrix::upload(M), dU = DeviceMatrix::upload(lr.U), dV = DeviceMatrix::upload(lr.V);
  check(slra_gemm(device_context(), 0, 0, M.rows(), n, lr.U.cols(), -1.0, dU.data(), dU.ld(), dV.data(), dV.ld(),
                  1.0, dM.data(), dM.ld()),
        "deterministic_error_diagnostic");
  double achieved = 0.0;
  check(slra_matrix_norm(device_context(), dM.data(), dM.ld(), M.rows(), n, 0, &achieved),
        "deterministic_error_diagnostic");
  return {bound, achieved};
}

// lra.cpp:88-127: sampled q x s entries of M - U V on the device, the
// estimate and its Wilson-Hilferty interval on the host
LraErrorEstimate posterior_error_estimate(const EntryOracle& M, const LowRankFactors& f, Index q, Index s, Rng& rng) {
  const Index m = M.rows(), n = M.cols();
  if (f.U.rows() != m || f.V.cols() != n) throw std::invalid_argument("posterior_error_estimate: factor shape mismatch");
  if (q < 1 || q > m || s < 1 || s > n || q * s < 2)
    throw std::invalid_argument("posterior_error_estimate: bad sample sizes");
  const IndexSet I(rng.distinct_indices(q, m), m);
  const IndexSet J(rng.distinct_indices(s, n), n);
  slra_ctx cx = device_context();
  const DeviceMatrix& dA = M.device();
  const Index l = f.U.cols();
  DevBuf<int64_t> dI(to64(I)), dJ(to64(J));
  DeviceMatrix Ms(q, s);
  check(slra_gather_block(cx, dA.data(), dA.ld(), m, n, dI.get(), q, dJ.get(), s, Ms.data(), Ms.ld()),
        "posterior_error_estimate");
  DevBuf<double> out(2);
  if (l > 0) {
    DeviceMatrix dU = DeviceMatrix::upload(f.U), dV = DeviceMatrix::upload(f.V), Us(q, l), Vs(l, s);
    check(slra_gather_rows(cx, dU.data(), dU.ld(), m, l, dI.get(), q, Us.data(), Us.ld()), "posterior_error_estimate");
    check(slra_gather_cols(cx, dV.data(), dV.ld(), l, n, dJ.get(), s, Vs.data(), Vs.ld()), "posterior_error_estimate");
    check(slra_lowrank_residual(cx, Ms.data(), Ms.ld(), q, s, Us.data(), Us.ld(), Vs.data(), Vs.ld(), l, out.get()),
          "posterior_error_estimate");
  } else {
    check(slra_lowrank_residual(cx, Ms.data(), Ms.ld(), q, s, nullptr, 1, nullptr, 1, 0, out.get()),
          "posterior_error_estimate");
  }
  M.count(static_cast<unsigned long long>(q * s));
  const double sumsq = out.download()[0];
  const double k = static_cast<double>(q * s);
  const double scale = static_cast<double>(m) * static_cast<double>(n);
  LraErrorEstimate est;
  est.estimate_frobenius = std::sqrt(scale * (sumsq / k));
  est.sample_rows = q;
  est.sample_cols = s;
  if (q * s >= 100) {
    auto chi2 = [k](double z) {
      const double t = 1.0 - 2.0 / (9.0 * k) + z * std::sqrt(2.0 / (9.0 * k));
      return k * t * t * t;
    };
    const double z975 = 1.959963984540054;
    est.ci_lo = std::sqrt(scale * sumsq / chi2(z975));
    est.ci_hi = std::sqrt(scale * sumsq / chi2(-z975));
    est.has_interval = true;
  } else {
    est.ci_lo = est.ci_hi = est.estimate_frobenius;
  }
  return est;
}

}  // namespace slra
