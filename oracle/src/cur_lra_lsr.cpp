// TEST INFRASTRUCTURE ONLY (see slra_oracle.hpp). Restates
// /root/reference/proj/src/cur.cpp, lra.cpp, lsr.cpp and the in-scope parts
// of testgen.cpp.
#include <algorithm>
#include <cmath>
#include <limits>

#include "slra_oracle.hpp"

namespace slra_oracle {

// ---------------------------------------------------------------- oracle gathers
// testgen.cpp:11-37
Matrix EntryOracle::rows_of(const IndexSet& I) const {
  Matrix out(I.size(), cols());
  for (Index t = 0; t < I.size(); ++t)
    for (Index j = 0; j < cols(); ++j) out(t, j) = entry(I[t], j);
  return out;
}
Matrix EntryOracle::cols_of(const IndexSet& J) const {
  Matrix out(rows(), J.size());
  for (Index t = 0; t < J.size(); ++t)
    for (Index i = 0; i < rows(); ++i) out(i, t) = entry(i, J[t]);
  return out;
}
Matrix EntryOracle::block(const IndexSet& I, const IndexSet& J) const {
  Matrix out(I.size(), J.size());
  for (Index s = 0; s < I.size(); ++s)
    for (Index t = 0; t < J.size(); ++t) out(s, t) = entry(I[s], J[t]);
  return out;
}
Matrix EntryOracle::dense() const {
  Matrix out(rows(), cols());
  for (Index i = 0; i < rows(); ++i)
    for (Index j = 0; j < cols(); ++j) out(i, j) = entry(i, j);
  return out;
}

// ---------------------------------------------------------------- cur.cpp
// cur.cpp:76-78: (C * U) * R, Eigen evaluates left to right.
Matrix cur_reconstruct(const Matrix& M, const CurDecomposition& c) {
  return matmul(matmul(select_cols(M, c.col_set), c.nucleus), select_rows(M, c.row_set));
}
// cur.cpp:80-82
double cur_evaluate(const Matrix& M, const CurDecomposition& c, NormKind norm) {
  return matrix_norm(sub(M, cur_reconstruct(M, c)), norm);
}
// cur.cpp:84-86
double t_factor(Index q, Index s, double h) {
  return std::sqrt(static_cast<double>(q - s) * static_cast<double>(s) * h * h + 1.0);
}

// cur.cpp:88-116
IndexSet maxvol_rows(const Matrix& A, double h, Index max_swaps) {
  const Index m = A.rows(), r = A.cols();
  if (r < 1 || m < r) throw std::invalid_argument("maxvol_rows: need m >= r >= 1");
  if (h < 1.0) throw std::invalid_argument("maxvol_rows: need h >= 1");
  if (max_swaps == 0) max_swaps = 4 * r;
  const Matrix At = A.transpose();
  ColPivQR init(At);
  std::vector<Index> I(static_cast<size_t>(r));
  for (Index t = 0; t < r; ++t) I[static_cast<size_t>(t)] = init.perm[static_cast<size_t>(t)];
  for (Index swap = 0; swap <= max_swaps; ++swap) {
    Matrix Gt(r, r);  // G^T, G = A[I,:]
    for (Index t = 0; t < r; ++t)
      for (Index c = 0; c < r; ++c) Gt(c, t) = A(I[static_cast<size_t>(t)], c);
    ColPivQR qr(Gt);
    qr.threshold = 1e-12;
    if (qr.rank() < r) throw SelectionFailure("maxvol_rows: singular pivot block");
    const Matrix X = qr.solve(At);  // r x m, B = X^T
    // B.cwiseAbs().maxCoeff(&bi,&bj): column-major traversal of B (m x r),
    // i.e. j outer, i inner; first strict maximum wins.
    Index bi = 0, bj = 0;
    double mx = -1;
    for (Index j = 0; j < r; ++j)
      for (Index i = 0; i < m; ++i) {
        const double v = std::abs(X(j, i));
        if (v > mx) {
          mx = v;
          bi = i;
          bj = j;
        }
      }
    if (mx <= h) break;
    if (swap == max_swaps) break;
    I[static_cast<size_t>(bj)] = bi;
  }
  return IndexSet(I, m);
}

// cur.cpp:118-135
IndexSet select_rows_spanning(const Matrix& A, Index count, double h) {
  const Index m = A.rows();
  if (count > m) throw std::invalid_argument("select_rows_spanning: count > rows");
  Matrix Q = thin_qr(A).first;
  const Index r = std::min(count, Q.cols());
  IndexSet base = maxvol_rows(Q.left_cols(r), h);
  if (count == r) return base;
  std::vector<Index> idx(base.begin(), base.end());
  std::vector<std::pair<double, Index>> rest;
  for (Index i = 0; i < m; ++i)
    if (!base.contains(i)) {
      double s = 0;
      for (Index j = 0; j < Q.cols(); ++j) s += Q(i, j) * Q(i, j);
      rest.emplace_back(std::sqrt(s), i);
    }
  // std::sort (not stable) in the reference; ties broken by index here.
  std::sort(rest.begin(), rest.end(), [](const auto& a, const auto& b) {
    return a.first > b.first || (a.first == b.first && a.second < b.second);
  });
  for (Index t = 0; t < count - r; ++t) idx.push_back(rest[static_cast<size_t>(t)].second);
  return IndexSet(std::move(idx), m);
}

// cur.cpp:137-162 (SVD nucleus; the qr_nucleus variant is out of scope)
CurDecomposition primitive_cur(const EntryOracle& M, IndexSet I, IndexSet J, Index r, bool qr_nucleus) {
  if (I.size() < r || J.size() < r || r < 1)
    throw std::invalid_argument("primitive_cur: need |I|, |J| >= r >= 1");
  Matrix G = M.block(I, J);
  CurDecomposition c;
  c.row_set = std::move(I);
  c.col_set = std::move(J);
  c.r = r;
  if (qr_nucleus) {  // cur.cpp:146-152: CompleteOrthogonalDecomposition, threshold 1e-10
    Index rank = 0;
    Matrix P = cod_pseudo_inverse(G, 1e-10, &rank);
    if (rank < r) throw GeneratorRankFailure("primitive_cur: generator rank below target");
    c.nucleus = std::move(P);
    return c;
  }
  Svd f = svd(G);
  if (f.sigma[0] <= 0 || f.sigma[static_cast<size_t>(r - 1)] <= 1e-10 * f.sigma[0])
    throw GeneratorRankFailure("primitive_cur: generator rank below target");
  // T_r diag(1/sigma_r) S_r^T
  const Index k = G.rows(), l = G.cols();
  Matrix TS(l, r);
  for (Index j = 0; j < r; ++j) {
    const double inv = 1.0 / f.sigma[static_cast<size_t>(j)];
    for (Index i = 0; i < l; ++i) TS(i, j) = f.T(i, j) * inv;
  }
  Matrix St(r, k);
  for (Index i = 0; i < k; ++i)
    for (Index j = 0; j < r; ++j) St(j, i) = f.S(i, j);
  c.nucleus = matmul(TS, St);
  return c;
}
CurDecomposition primitive_cur(const Matrix& M, IndexSet I, IndexSet J, Index r, bool qr_nucleus) {
  DenseOracle o(M);
  return primitive_cur(o, std::move(I), std::move(J), r, qr_nucleus);
}

namespace {
// cur.cpp:192-197
double block_volume(const Matrix& Q, const IndexSet& I) {
  if (I.size() != Q.cols()) return 0;
  return determinant_abs(select_rows(Q, I));
}
}  // namespace

// cur.cpp:201-255
std::pair<CurDecomposition, CaTrace> cross_approx(const EntryOracle& M, Index r, Index k, Index l,
                                                  IndexSet init_rows, int loops, double h,
                                                  std::optional<double> stop_tol, Rng& rng) {
  const Index m = M.rows(), n = M.cols();
  if (k < r || l < r || r < 1) throw std::invalid_argument("cross_approx: need k, l >= r >= 1");
  if (loops < 1) throw std::invalid_argument("cross_approx: need loops >= 1");
  IndexSet I = (init_rows.size() == k && init_rows.bound() == m) ? std::move(init_rows)
                                                                 : IndexSet(rng.distinct_indices(k, m), m);
  IndexSet J;
  CaTrace trace;
  for (int loop = 0; loop < loops; ++loop) {
    Matrix R = M.rows_of(I);
    const Matrix Rt = R.transpose();
    J = select_rows_spanning(Rt, l, h);
    {
      CaStep st;
      st.horizontal = false;
      st.rows.assign(I.begin(), I.end());
      st.cols.assign(J.begin(), J.end());
      st.volume_proxy = block_volume(thin_qr(Rt).first, J);
      trace.steps.push_back(std::move(st));
    }
    Matrix C = M.cols_of(J);
    I = select_rows_spanning(C, k, h);
    {
      CaStep st;
      st.horizontal = true;
      st.rows.assign(I.begin(), I.end());
      st.cols.assign(J.begin(), J.end());
      st.volume_proxy = block_volume(thin_qr(C).first, I);
      if (stop_tol) {
        try {
          CurDecomposition probe = primitive_cur(M, I, J, r);
          LowRankFactors f;
          f.U = matmul(M.cols_of(J), probe.nucleus);
          f.V = M.rows_of(I);
          f.target_rank = r;
          const Index q = std::min<Index>(20, m), s = std::min<Index>(20, n);
          st.error_estimate = posterior_error_estimate(M, f, q, s, rng).estimate_frobenius;
        } catch (const GeneratorRankFailure&) {
          st.error_estimate.reset();
        }
      }
      const bool stop = stop_tol && st.error_estimate && *st.error_estimate <= *stop_tol;
      trace.steps.push_back(std::move(st));
      if (stop) break;
    }
  }
  return {primitive_cur(M, std::move(I), std::move(J), r), std::move(trace)};
}

// ---------------------------------------------------------------- lra.cpp
namespace {
// lra.cpp:14-27
Matrix range_basis(const Matrix& M, const SketchOperator& H, Index r, RangeVariant variant) {
  if (H.rows() != M.cols()) throw std::invalid_argument("range_finder: H rows != n");
  const Index l = H.cols();
  if (r < 1 || r > l) throw std::invalid_argument("range_finder: need 1 <= r <= l");
  Matrix MH = apply(H, M, Side::Right);
  if (numerical_rank(MH, 1e-10, RankMode::Relative) < r)
    throw RangeFailure("range_finder: sketch M H has numerical rank below target");
  if (variant == RangeVariant::BasisQr) return thin_qr(MH).first;
  Svd f = svd(MH);
  Matrix U(MH.rows(), r);
  for (Index j = 0; j < r; ++j)
    for (Index i = 0; i < MH.rows(); ++i) U(i, j) = f.S(i, j) * f.sigma[static_cast<size_t>(j)];
  return U;
}
}  // namespace

// lra.cpp:31-39
LowRankFactors range_finder(const Matrix& M, const SketchOperator& H, Index r, RangeVariant variant) {
  LowRankFactors out;
  out.U = range_basis(M, H, r, variant);
  out.V = (variant == RangeVariant::BasisQr) ? matmul_tn(out.U, M) : matmul(pseudo_inverse(out.U), M);
  out.target_rank = r;
  return out;
}

// lra.cpp:41-52: U as range_finder's, V = (F U)^+ (F M); PremultRankFailure
// when numerical_rank(F U, 1e-10, Relative) < r.
LowRankFactors lra_premult(const Matrix& M, const SketchOperator& F, const SketchOperator& H, Index r,
                           RangeVariant variant) {
  if (F.cols() != M.rows()) throw std::invalid_argument("lra_premult: F cols != m");
  LowRankFactors out;
  out.U = range_basis(M, H, r, variant);
  const Matrix FU = apply(F, out.U, Side::Left);
  if (numerical_rank(FU, 1e-10, RankMode::Relative) < r)
    throw PremultRankFailure("lra_premult: F U has numerical rank below target");
  out.V = matmul(pseudo_inverse(FU), apply(F, M, Side::Left));
  out.target_rank = r;
  return out;
}

// lra.cpp:54-63
LowRankFactors two_stage_truncate(const LowRankFactors& f, Index r) {
  if (r < 1 || r > f.U.cols()) throw std::invalid_argument("two_stage_truncate: need 1 <= r <= l");
  auto [Q, R] = thin_qr(f.U);
  Svd core = svd(matmul(R, f.V));
  LowRankFactors out;
  Matrix Sr(core.S.rows(), r);
  for (Index j = 0; j < r; ++j)
    for (Index i = 0; i < core.S.rows(); ++i) Sr(i, j) = core.S(i, j) * core.sigma[static_cast<size_t>(j)];
  out.U = matmul(Q, Sr);
  out.V = core.T.left_cols(r).transpose();
  out.target_rank = r;
  return out;
}

// lra.cpp:88-127
LraErrorEstimate posterior_error_estimate(const EntryOracle& M, const LowRankFactors& f, Index q,
                                          Index s, Rng& rng) {
  const Index m = M.rows(), n = M.cols();
  if (f.U.rows() != m || f.V.cols() != n)
    throw std::invalid_argument("posterior_error_estimate: factor shape mismatch");
  if (q < 1 || q > m || s < 1 || s > n || q * s < 2)
    throw std::invalid_argument("posterior_error_estimate: bad sample sizes");
  const IndexSet I(rng.distinct_indices(q, m), m);
  const IndexSet J(rng.distinct_indices(s, n), n);
  double sumsq = 0;
  for (Index a = 0; a < q; ++a)
    for (Index b = 0; b < s; ++b) {
      double dot = 0;
      for (Index t = 0; t < f.U.cols(); ++t) dot += f.U(I[a], t) * f.V(t, J[b]);
      const double e = M.entry(I[a], J[b]) - dot;
      sumsq += e * e;
    }
  const double k = static_cast<double>(q * s);
  const double mean_sq = sumsq / k;
  const double scale = static_cast<double>(m) * static_cast<double>(n);
  LraErrorEstimate est;
  est.estimate_frobenius = std::sqrt(scale * mean_sq);
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

// ---------------------------------------------------------------- lsr.cpp
namespace {
void validate(const LsrProblem& p) {  // lsr.cpp:13-17
  if (p.A.rows() <= p.A.cols() || p.A.cols() < 1) throw std::invalid_argument("lsr: need m > d >= 1");
  if (static_cast<Index>(p.b.size()) != p.A.rows()) throw std::invalid_argument("lsr: b length mismatch");
}
Matrix as_col(const Vector& b) {
  Matrix B(static_cast<Index>(b.size()), 1);
  std::copy(b.begin(), b.end(), B.v.begin());
  return B;
}
}  // namespace

// lsr.cpp:21-24
Vector solve_exact(const LsrProblem& p) {
  validate(p);
  Matrix x = matmul(pseudo_inverse(p.A), as_col(p.b));
  return x.v;
}
// lsr.cpp:26-28
double residual_norm(const LsrProblem& p, const Vector& x) {
  Matrix Ax = matmul(p.A, as_col(x));
  double s = 0;
  for (Index i = 0; i < p.A.rows(); ++i) {
    const double e = Ax(i, 0) - p.b[static_cast<size_t>(i)];
    s += e * e;
  }
  return std::sqrt(s);
}
// lsr.cpp:30-35
double residual_ratio(const LsrProblem& p, const Vector& x_hat) {
  const double opt = residual_norm(p, solve_exact(p));
  double bn = 0;
  for (double x : p.b) bn += x * x;
  if (opt < 1e-14 * std::sqrt(bn)) return std::numeric_limits<double>::infinity();
  return residual_norm(p, x_hat) / opt;
}
// lsr.cpp:37-67
LsrReport sketch_solve(const LsrProblem& p, const SketchOperator& F, bool with_true_residual) {
  validate(p);
  const Index d = p.A.cols(), m = p.A.rows();
  if (F.cols() != m) throw std::invalid_argument("sketch_solve: F cols != m");
  if (F.rows() <= d) throw std::invalid_argument("sketch_solve: need k > d");
  Matrix W(m, d + 1);
  std::copy(p.A.v.begin(), p.A.v.end(), W.v.begin());
  std::copy(p.b.begin(), p.b.end(), W.v.begin() + m * d);
  Matrix Mw = F.apply(W);
  const Index k = Mw.rows();
  Matrix FA = Mw.left_cols(d);
  Matrix Fb(k, 1);
  std::copy(Mw.col(d), Mw.col(d) + k, Fb.v.begin());
  ColPivQR qr(FA);
  qr.threshold = 1e-10;
  if (qr.rank() < d) throw SketchRankFailure("sketch_solve: sketched matrix FA is rank deficient");
  LsrReport rep;
  Matrix x = qr.solve(Fb);
  rep.x_hat = x.v;
  Matrix FAx = matmul(FA, x);
  double s = 0;
  for (Index i = 0; i < k; ++i) {
    const double e = FAx(i, 0) - Fb(i, 0);
    s += e * e;
  }
  rep.sketched_residual = std::sqrt(s);
  rep.k = F.rows();
  if (with_true_residual) {
    rep.true_residual = residual_norm(p, rep.x_hat);
    rep.ratio = residual_ratio(p, rep.x_hat);
  }
  return rep;
}

// lsr.cpp:69-113: sketch-and-solve with re-randomised retries, each solution
// validated against an independently drawn sketch of the same shape.
LsrReport solve_with_retries(const LsrProblem& p, OpPtr base_F, const std::vector<OpPtr>& q_family,
                             int max_retries, double accept_tol, Rng& rng) {
  validate(p);
  const Index m = p.A.rows();
  LsrReport best;
  double best_score = std::numeric_limits<double>::infinity();
  bool have_best = false;
  for (int attempt = 0; attempt <= max_retries; ++attempt) {
    OpPtr F = base_F;
    if (attempt > 0) {
      OpPtr Q = q_family.empty() ? gen_permutation(m, rng)
                                 : q_family[static_cast<size_t>((attempt - 1) % static_cast<int>(q_family.size()))];
      F = make_product({base_F, Q});
    }
    LsrReport rep;
    try {
      rep = sketch_solve(p, *F);
    } catch (const SketchRankFailure&) {
      continue;
    }
    rep.attempts = attempt + 1;
    OpPtr Fv = make_product({base_F, gen_permutation(m, rng)});
    const Matrix VA = Fv->apply(p.A);
    Matrix bm(m, 1);
    for (Index i = 0; i < m; ++i) bm(i, 0) = p.b[static_cast<size_t>(i)];
    const Matrix vb = Fv->apply(bm);
    double rv = 0, vn = 0;
    for (Index i = 0; i < VA.rows(); ++i) {
      double s = 0;
      for (Index j = 0; j < VA.cols(); ++j) s += VA(i, j) * rep.x_hat[static_cast<size_t>(j)];
      const double e = s - vb(i, 0);
      rv += e * e;
      vn += vb(i, 0) * vb(i, 0);
    }
    const double r_val = std::sqrt(rv);
    const double score = r_val / std::max(rep.sketched_residual, 1e-300);
    const bool ok = r_val <= 1e-12 * std::sqrt(vn) || score <= accept_tol;
    rep.validated = ok;
    if (ok) return rep;
    if (score < best_score) {
      best_score = score;
      best = rep;
      have_best = true;
    }
  }
  if (!have_best) throw SketchRankFailure("solve_with_retries: all attempts rank deficient");
  best.validated = false;
  return best;
}

// ---------------------------------------------------------------- testgen.cpp
Matrix random_orthonormal(Index rows, Index cols, Rng& rng) {  // testgen.cpp:41-43
  return thin_qr(rng.gaussian_matrix(rows, cols)).first;
}
Matrix gen_svd_profile(Index n, Index r, Rng& rng) {  // testgen.cpp:100-108
  if (r >= n) throw std::invalid_argument("gen_svd_profile: need r < n");
  Matrix S = random_orthonormal(n, n, rng);
  Matrix T = random_orthonormal(n, n, rng);
  for (Index j = 0; j < n; ++j) {
    const double sj = (j < r) ? 1.0 / static_cast<double>(j + 1) : 1e-10;
    for (Index i = 0; i < n; ++i) S(i, j) *= sj;
  }
  return matmul(S, T.transpose());
}
Matrix gen_factor_gaussian(Index m, Index n, Index r, double noise, Rng& rng) {  // :110-115
  if (r > std::min(m, n)) throw std::invalid_argument("gen_factor_gaussian: r too large");
  Matrix G1 = rng.gaussian_matrix(m, r);
  Matrix G2 = rng.gaussian_matrix(r, n);
  Matrix M = matmul(G1, G2);
  if (noise != 0) {
    Matrix N = rng.gaussian_matrix(m, n);
    for (Index t = 0; t < M.size(); ++t) M.v[static_cast<size_t>(t)] += noise * N.v[static_cast<size_t>(t)];
  }
  return M;
}
LsrProblem gen_lsr_gaussian(Index m, Index n, double noise, Rng& rng) {  // :159-193
  if (m <= n) throw std::invalid_argument("gen_lsr_family: need m > n");
  LsrProblem p;
  p.A = rng.gaussian_matrix(m, n);
  Vector x0 = rng.gaussian_vector(n);
  Vector e = rng.gaussian_vector(m);
  Matrix Ax = matmul(p.A, as_col(x0));
  p.b.resize(static_cast<size_t>(m));
  for (Index i = 0; i < m; ++i) p.b[static_cast<size_t>(i)] = Ax(i, 0) + noise * e[static_cast<size_t>(i)];
  return p;
}

}  // namespace slra_oracle
