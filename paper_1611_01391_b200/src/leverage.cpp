// Leverage-score CUR (/root/reference/proj/src/leverage.cpp:12-196 and
// lra_to_top_svd, cur.cpp:257-276) over the C-ABI. The matrix and every
// factor stay in HBM: SVDs (one-CTA or multi-CTA Jacobi), score vectors
// (row squared norms), gathers, diagonal rescalings and the truncated
// pseudo-inverse nuclei are device passes. The draws themselves
// (categorical / Bernoulli over the score vector) are host logic on the
// caller's Rng, in the reference's order, so the index sets match.
#include "slra/leverage.hpp"

#include <algorithm>
#include <cmath>
#include <map>

#include "slra/devbuf.hpp"
#include "slra/errors.hpp"

namespace slra {

namespace {

std::vector<int64_t> to64(const std::vector<Index>& v) { return std::vector<int64_t>(v.begin(), v.end()); }

struct DevSvd {
  DeviceMatrix S, T;
  DevBuf<double> sigma;
  std::vector<double> hsig;
  Index p = 0;
};

DevSvd dsvd(const double* A, Index lda, Index m, Index n) {
  DevSvd f;
  f.p = std::min(m, n);
  f.S = DeviceMatrix(m, f.p);
  f.T = DeviceMatrix(n, f.p);
  f.sigma = DevBuf<double>(static_cast<size_t>(f.p));
  check(slra_svd(device_context(), A, lda, m, n, f.S.data(), f.S.ld(), f.sigma.get(), f.T.data(), f.T.ld()), "svd");
  f.hsig = f.sigma.download();
  return f;
}

// sigma(r-1) <= 1e-10 sigma(0) -> GeneratorRankFailure (leverage.cpp:101-102, 111-112, 121-122, 127-128)
void check_rank(const std::vector<double>& s, Index r, const char* what) {
  if (s.empty() || static_cast<Index>(s.size()) < r || s[0] <= 0 || s[static_cast<size_t>(r - 1)] <= 1e-10 * s[0])
    throw GeneratorRankFailure(what);
}

// svd_leverage_scores (leverage.cpp:12-23) of the n x r device factor T
// (ld ldt): orthonormality ||T^T T - I||_2 <= 1e-8 (one GEMM + one SVD of
// r x r), then p = rowwise squared norms / r.
LeverageScores scores_device(const double* T, Index ldt, Index n, Index r, double beta) {
  if (r < 1 || n < r) throw std::invalid_argument("svd_leverage_scores: bad shape");
  if (beta <= 0 || beta > 1) throw std::invalid_argument("svd_leverage_scores: beta in (0,1]");
  slra_ctx cx = device_context();
  Matrix I(r, r);
  for (Index i = 0; i < r; ++i) I(i, i) = 1.0;
  DeviceMatrix G = DeviceMatrix::upload(I);
  check(slra_gemm(cx, 1, 0, r, r, n, 1.0, T, ldt, T, ldt, -1.0, G.data(), G.ld()), "svd_leverage_scores");
  double dev = 0.0;
  check(slra_matrix_norm(cx, G.data(), G.ld(), r, r, 0, &dev), "svd_leverage_scores");
  if (dev > 1e-8) throw std::invalid_argument("svd_leverage_scores: columns not orthonormal");
  DevBuf<double> p(static_cast<size_t>(n));
  check(slra_row_sqnorms(cx, T, ldt, n, r, static_cast<double>(r), p.get()), "svd_leverage_scores");
  LeverageScores s;
  s.p = p.download();
  s.beta = beta;
  s.r = r;
  return s;
}

// T_r diag(1/sigma_r) S_r^T (Eigen: (T_r * inv.asDiagonal()) * S_r^T)
DeviceMatrix truncated_pinv(const DevSvd& g, Index r) {
  slra_ctx cx = device_context();
  const Index n = g.T.rows(), m = g.S.rows();
  std::vector<double> inv(static_cast<size_t>(r));
  for (Index j = 0; j < r; ++j) inv[static_cast<size_t>(j)] = 1.0 / g.hsig[static_cast<size_t>(j)];
  DevBuf<double> dinv(inv);
  DeviceMatrix TS(n, r), P(n, m);
  check(slra_scale_rows_cols(cx, g.T.data(), g.T.ld(), n, r, nullptr, dinv.get(), TS.data(), TS.ld()), "pinv");
  check(slra_gemm(cx, 0, 1, n, m, r, 1.0, TS.data(), TS.ld(), g.S.data(), g.S.ld(), 0.0, P.data(), P.ld()), "pinv");
  return P;
}

// leverage.cpp:76-86
SampleRescale draw(const LeverageScores& scores, Index l, SampleMode mode, Rng& rng) {
  if (mode == SampleMode::Exactly) return sample_exactly(scores, l, rng);
  for (int attempt = 0; attempt < 8; ++attempt) {
    try {
      return sample_expected(scores, l, rng);
    } catch (const EmptySample&) {
    }
  }
  throw EmptySample("cur_via_leverage: expected-mode sampling stayed empty after 8 tries");
}

}  // namespace

LeverageScores svd_leverage_scores(const Matrix& T, double beta) {
  if (T.cols() < 1 || T.rows() < T.cols()) throw std::invalid_argument("svd_leverage_scores: bad shape");
  DeviceMatrix dT = DeviceMatrix::upload(T);
  return scores_device(dT.data(), dT.ld(), T.rows(), T.cols(), beta);
}

// leverage.cpp:25-41 (host draws over the score vector)
SampleRescale sample_exactly(const LeverageScores& scores, Index l, Rng& rng) {
  if (l < 1) throw std::invalid_argument("sample_exactly: l >= 1");
  const Index n = static_cast<Index>(scores.p.size());
  double total = 0;
  for (double x : scores.p) total += x;
  SampleRescale out;
  out.d.assign(static_cast<size_t>(l), 0.0);
  for (Index t = 0; t < l; ++t) {
    double u = rng.uniform() * total;
    Index i = 0;
    while (i + 1 < n && u > scores.p[static_cast<size_t>(i)]) u -= scores.p[static_cast<size_t>(i)], ++i;
    while (i > 0 && scores.p[static_cast<size_t>(i)] <= 0) --i;
    out.indices.push_back(i);
    out.d[static_cast<size_t>(t)] = 1.0 / std::sqrt(static_cast<double>(l) * scores.p[static_cast<size_t>(i)]);
  }
  return out;
}

// leverage.cpp:43-58
SampleRescale sample_expected(const LeverageScores& scores, Index l, Rng& rng) {
  if (l < 1) throw std::invalid_argument("sample_expected: l >= 1");
  SampleRescale out;
  for (size_t j = 0; j < scores.p.size(); ++j) {
    const double q = std::min(1.0, static_cast<double>(l) * scores.p[j]);
    if (q > 0 && rng.uniform() < q) {
      out.indices.push_back(static_cast<Index>(j));
      out.d.push_back(1.0 / std::min(1.0, std::sqrt(static_cast<double>(l) * scores.p[j])));
    }
  }
  if (out.indices.empty()) throw EmptySample("sample_expected: no columns kept");
  return out;
}

// leverage.cpp:60-72
SampleRescale collapse_duplicates(const SampleRescale& s) {
  std::map<Index, double> acc;
  for (size_t t = 0; t < s.indices.size(); ++t) acc[s.indices[t]] += s.d[t] * s.d[t];
  SampleRescale out;
  for (const auto& [i, w2] : acc) {
    out.indices.push_back(i);
    out.d.push_back(std::sqrt(w2));
  }
  return out;
}

// leverage.cpp:88-149
CurDecomposition cur_via_leverage(const EntryOracle& M, Index r, Index k, Index l, double beta, double beta_bar,
                                  SampleMode mode, const std::optional<LeverageScores>& scores, Rng& rng,
                                  bool plain_nucleus) {
  const Index m = M.rows(), n = M.cols();
  if (r < 1 || k < r || l < r) throw std::invalid_argument("cur_via_leverage: need k, l >= r");
  slra_ctx cx = device_context();
  const DeviceMatrix& dA = M.device();
  LeverageScores col_scores;
  if (scores) {
    col_scores = *scores;
    if (static_cast<Index>(col_scores.p.size()) != n)
      throw std::invalid_argument("cur_via_leverage: scores length != n");
  } else {
    const DevSvd f = dsvd(dA.data(), dA.ld(), m, n);
    M.count(static_cast<unsigned long long>(m * n));
    check_rank(f.hsig, r, "cur_via_leverage: input rank below target");
    col_scores = scores_device(f.T.data(), f.T.ld(), n, r, beta);
  }
  // columns, then the rescaled column factor, then rows
  const SampleRescale cs = collapse_duplicates(draw(col_scores, l, mode, rng));
  const Index lc = static_cast<Index>(cs.indices.size());
  DevBuf<int64_t> dJ(to64(cs.indices));
  DevBuf<double> dcs(cs.d);
  DeviceMatrix CD(m, lc);
  check(slra_gather_cols(cx, dA.data(), dA.ld(), m, n, dJ.get(), lc, CD.data(), CD.ld()), "cur_via_leverage");
  check(slra_scale_rows_cols(cx, CD.data(), CD.ld(), m, lc, nullptr, dcs.get(), CD.data(), CD.ld()),
        "cur_via_leverage");
  M.count(static_cast<unsigned long long>(m * lc));
  const DevSvd cf = dsvd(CD.data(), CD.ld(), m, lc);
  check_rank(cf.hsig, r, "cur_via_leverage: sampled column factor rank below target");
  const LeverageScores row_scores = scores_device(cf.S.data(), cf.S.ld(), m, r, beta_bar);
  const SampleRescale rs = collapse_duplicates(draw(row_scores, k, mode, rng));
  const Index kr = static_cast<Index>(rs.indices.size());
  DevBuf<int64_t> dI(to64(rs.indices));
  DevBuf<double> drs(rs.d);
  DeviceMatrix G(kr, lc);
  check(slra_gather_block(cx, dA.data(), dA.ld(), m, n, dI.get(), kr, dJ.get(), lc, G.data(), G.ld()),
        "cur_via_leverage");
  M.count(static_cast<unsigned long long>(kr * lc));
  CurDecomposition c;
  c.r = r;
  if (plain_nucleus) {
    const DevSvd g = dsvd(G.data(), G.ld(), kr, lc);
    check_rank(g.hsig, r, "cur_via_leverage: generator rank below target");
    c.nucleus = truncated_pinv(g, r).download();
  } else {
    check(slra_scale_rows_cols(cx, G.data(), G.ld(), kr, lc, drs.get(), dcs.get(), G.data(), G.ld()),
          "cur_via_leverage");
    const DevSvd g = dsvd(G.data(), G.ld(), kr, lc);
    check_rank(g.hsig, r, "cur_via_leverage: rescaled generator rank below target");
    DeviceMatrix P = truncated_pinv(g, r);  // lc x kr
    check(slra_scale_rows_cols(cx, P.data(), P.ld(), lc, kr, dcs.get(), drs.get(), P.data(), P.ld()),
          "cur_via_leverage");
    c.nucleus = P.download();
  }
  c.row_set = IndexSet(rs.indices, m);
  c.col_set = IndexSet(cs.indices, n);
  return c;
}

// cur.cpp:257-276 with W = I (the LowRankFactors overload)
Svd lra_to_top_svd(const LowRankFactors& f, Index r) {
  const Index l = f.U.cols(), m = f.U.rows(), n = f.V.cols();
  if (f.V.rows() != l) throw std::invalid_argument("lra_to_top_svd: inner dimension mismatch");
  if (r < 1 || r > l) throw std::invalid_argument("lra_to_top_svd: bad rank");
  slra_ctx cx = device_context();
  DeviceMatrix dU = DeviceMatrix::upload(f.U), dV = DeviceMatrix::upload(f.V), Vt(n, l);
  DeviceMatrix QA(m, l), RA(l, l), QB(n, l), RB(l, l), core(l, l);
  check(slra_thin_qr(cx, dU.data(), dU.ld(), m, l, QA.data(), QA.ld(), RA.data(), RA.ld()), "lra_to_top_svd");
  check(slra_transpose(cx, dV.data(), dV.ld(), l, n, Vt.data(), Vt.ld()), "lra_to_top_svd");
  check(slra_thin_qr(cx, Vt.data(), Vt.ld(), n, l, QB.data(), QB.ld(), RB.data(), RB.ld()), "lra_to_top_svd");
  // RA W RB^T with W = I: RA * I is exact
  check(slra_gemm(cx, 0, 1, l, l, l, 1.0, RA.data(), RA.ld(), RB.data(), RB.ld(), 0.0, core.data(), core.ld()),
        "lra_to_top_svd");
  const DevSvd g = dsvd(core.data(), core.ld(), l, l);
  if (g.hsig[0] <= 0 || g.hsig[static_cast<size_t>(r - 1)] <= 1e-13 * g.hsig[0])
    throw GeneratorRankFailure("lra_to_top_svd: core rank below target");
  DeviceMatrix S(m, r), T(n, r);
  check(slra_gemm(cx, 0, 0, m, r, l, 1.0, QA.data(), QA.ld(), g.S.data(), g.S.ld(), 0.0, S.data(), S.ld()),
        "lra_to_top_svd");
  check(slra_gemm(cx, 0, 0, n, r, l, 1.0, QB.data(), QB.ld(), g.T.data(), g.T.ld(), 0.0, T.data(), T.ld()),
        "lra_to_top_svd");
  Svd out;
  out.S = S.download();
  out.sigma.assign(g.hsig.begin(), g.hsig.begin() + r);
  out.T = T.download();
  return out;
}

// leverage.cpp:151-157
CurDecomposition refine_lra(const EntryOracle& M, const LowRankFactors& crude, Index r, Index k, Index l, Rng& rng) {
  if (crude.target_rank < r) throw std::invalid_argument("refine_lra: crude rank below target");
  const Svd top = lra_to_top_svd(crude, r);
  const LeverageScores scores = svd_leverage_scores(top.T, 1.0);
  return cur_via_leverage(M, r, k, l, 1.0, 1.0, SampleMode::Exactly, scores, rng);
}

LeverageScores uniform_scores(Index n) {  // leverage.cpp:159-166
  if (n < 1) throw std::invalid_argument("uniform_scores: n >= 1");
  LeverageScores s;
  s.p.assign(static_cast<size_t>(n), 1.0 / static_cast<double>(n));
  s.beta = 1.0;
  s.r = 1;
  return s;
}

// leverage.cpp:168-180 (an evaluator): scores of G / sqrt(n) on the device
// against the column-norm surrogate, max gap over the n columns.
double gaussian_score_gap(const Matrix& G) {
  const Index r = G.rows(), n = G.cols();
  if (r > n) throw std::invalid_argument("gaussian_score_gap: need r <= n");
  slra_ctx cx = device_context();
  Matrix Gs(r, n);
  const double sn = std::sqrt(static_cast<double>(n));
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < r; ++i) Gs(i, j) = G(i, j) / sn;
  DeviceMatrix dGs = DeviceMatrix::upload(Gs), dG = DeviceMatrix::upload(G), Gt(n, r);
  const DevSvd f = dsvd(dGs.data(), dGs.ld(), r, n);
  DevBuf<double> p(static_cast<size_t>(n)), q(static_cast<size_t>(n));
  check(slra_row_sqnorms(cx, f.T.data(), f.T.ld(), n, r, static_cast<double>(r), p.get()), "gaussian_score_gap");
  check(slra_transpose(cx, dG.data(), dG.ld(), r, n, Gt.data(), Gt.ld()), "gaussian_score_gap");
  check(slra_row_sqnorms(cx, Gt.data(), Gt.ld(), n, r, static_cast<double>(n) * static_cast<double>(r), q.get()),
        "gaussian_score_gap");
  const std::vector<double> hp = p.download(), hq = q.download();
  double gap = 0;
  for (Index j = 0; j < n; ++j) gap = std::max(gap, std::abs(hp[static_cast<size_t>(j)] - hq[static_cast<size_t>(j)]));
  return gap;
}

double sample_bound_quadratic(Index r, double eps, double beta) {  // leverage.cpp:182-184
  return 3200.0 * static_cast<double>(r) * static_cast<double>(r) / (eps * eps * beta);
}
double sample_bound_loglinear(Index r, double eps, double beta, double cbar) {  // :186-188
  return cbar * static_cast<double>(r) * std::log(static_cast<double>(r)) / (eps * eps * beta);
}
double epsilon_for_sample(Index r, Index l, double delta) {  // :190-194
  return std::sqrt(4.0 * static_cast<double>(r) * std::log(2.0 * static_cast<double>(r) / delta) /
                   static_cast<double>(l));
}

}  // namespace slra
