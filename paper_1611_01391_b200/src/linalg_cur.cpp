// Host entry points of linalg.hpp / cur.hpp / lra.hpp: reference signatures
// (/root/reference/proj/include/slra/{linalg,cur,lra}.hpp) over the C-ABI.
// Every numeric result is computed on the device; the host only moves
// operands, builds index sets and rethrows typed failures.
#include <algorithm>
#include <cmath>

#include "slra/cur.hpp"
#include "slra/devbuf.hpp"
#include "slra/errors.hpp"
#include "slra/lra.hpp"

namespace slra {

namespace {
std::vector<int64_t> to64(const IndexSet& s) { return std::vector<int64_t>(s.begin(), s.end()); }
}  // namespace

// ---------------------------------------------------------------- linalg
Matrix matmul(const Matrix& A, const Matrix& B) {  // linalg.cpp:63-66
  if (A.cols() != B.rows()) throw std::invalid_argument("matmul: dimension mismatch");
  DeviceMatrix dA = DeviceMatrix::upload(A), dB = DeviceMatrix::upload(B), dC(A.rows(), B.cols());
  check(slra_gemm(device_context(), 0, 0, A.rows(), B.cols(), A.cols(), 1.0, dA.data(), dA.ld(), dB.data(), dB.ld(),
                  0.0, dC.data(), dC.ld()),
        "slra_gemm");
  return dC.download();
}

std::pair<Matrix, Matrix> thin_qr(const Matrix& A) {  // linalg.cpp:67-79
  if (A.rows() < A.cols()) throw std::invalid_argument("thin_qr: rows < cols");
  DeviceMatrix dA = DeviceMatrix::upload(A), dQ(A.rows(), A.cols()), dR(A.cols(), A.cols());
  check(slra_thin_qr(device_context(), dA.data(), dA.ld(), A.rows(), A.cols(), dQ.data(), dQ.ld(), dR.data(), dR.ld()),
        "slra_thin_qr");
  return {dQ.download(), dR.download()};
}

Svd svd(const Matrix& A) {  // linalg.cpp:81-98
  const Index p = std::min(A.rows(), A.cols());
  DeviceMatrix dA = DeviceMatrix::upload(A), dS(A.rows(), p), dT(A.cols(), p);
  DevBuf<double> sig(static_cast<size_t>(p));
  check(slra_svd(device_context(), dA.data(), dA.ld(), A.rows(), A.cols(), dS.data(), dS.ld(), sig.get(), dT.data(),
                 dT.ld()),
        "slra_svd");
  return Svd{dS.download(), sig.download(), dT.download()};
}

Matrix pseudo_inverse(const Matrix& A, double rank_tol) {  // linalg.cpp:111-121
  DeviceMatrix dA = DeviceMatrix::upload(A), dP(A.cols(), A.rows());
  int64_t rho = 0;
  check(slra_pinv(device_context(), dA.data(), dA.ld(), A.rows(), A.cols(), rank_tol, dP.data(), dP.ld(), &rho),
        "slra_pinv");
  return dP.download();
}

Index numerical_rank(const Matrix& A, double tol, RankMode mode) {  // linalg.cpp:123-132
  if (tol <= 0) throw std::invalid_argument("numerical_rank: tol must be positive");
  const Svd f = svd(A);
  if (f.sigma.empty()) return 0;
  const double cut = (mode == RankMode::Absolute) ? tol : tol * f.sigma[0];
  Index count = 0;
  for (double s : f.sigma) count += s > cut;
  return count;
}

double matrix_norm(const Matrix& A, NormKind kind) {  // linalg.cpp:134-151 on the device
  if (A.rows() == 0 || A.cols() == 0) return 0.0;
  DeviceMatrix dA = DeviceMatrix::upload(A);
  double v = 0.0;
  const int k = kind == NormKind::Spectral ? 0 : kind == NormKind::Frobenius ? 1 : 2;
  check(slra_matrix_norm(device_context(), dA.data(), dA.ld(), A.rows(), A.cols(), k, &v), "matrix_norm");
  return v;
}
double spectral_norm(const Matrix& A) { return matrix_norm(A, NormKind::Spectral); }
double chebyshev_norm(const Matrix& A) { return matrix_norm(A, NormKind::Chebyshev); }

double frobenius_norm(const Matrix& A) {  // linalg.cpp:139, one device pass
  DeviceMatrix dA = DeviceMatrix::upload(A);
  DevBuf<double> out(2);
  check(slra_lowrank_residual(device_context(), dA.data(), dA.ld(), A.rows(), A.cols(), nullptr, 1, nullptr, 1, 0,
                              out.get()),
        "slra_lowrank_residual");
  return std::sqrt(out.download()[1]);
}

// ---------------------------------------------------------------- cur
double t_factor(Index q, Index s, double h) {  // cur.cpp:84-86
  return std::sqrt(static_cast<double>(q - s) * static_cast<double>(s) * h * h + 1.0);
}

IndexSet maxvol_rows(const Matrix& A, double h, Index max_swaps) {  // cur.cpp:88-116
  const Index m = A.rows(), r = A.cols();
  if (r < 1 || m < r) throw std::invalid_argument("maxvol_rows: need m >= r >= 1");
  if (h < 1.0) throw std::invalid_argument("maxvol_rows: need h >= 1");
  DeviceMatrix dA = DeviceMatrix::upload(A);
  DevBuf<int64_t> idx(static_cast<size_t>(r));
  check(slra_maxvol_rows(device_context(), dA.data(), dA.ld(), m, r, h, max_swaps, idx.get()), "maxvol_rows");
  auto v = idx.download();
  return IndexSet(std::vector<Index>(v.begin(), v.end()), m);
}

IndexSet select_rows_spanning(const Matrix& A, Index count, double h) {  // cur.cpp:118-135
  const Index m = A.rows();
  if (count > m) throw std::invalid_argument("select_rows_spanning: count > rows");
  DeviceMatrix dA = DeviceMatrix::upload(A);
  DevBuf<int64_t> idx(static_cast<size_t>(count));
  check(slra_select_rows_spanning(device_context(), dA.data(), dA.ld(), m, A.cols(), count, h, idx.get(), nullptr),
        "select_rows_spanning");
  auto v = idx.download();
  return IndexSet(std::vector<Index>(v.begin(), v.end()), m);
}

// factored nucleus U = tsig * sr^T from the device buffers (first r columns)
static void set_factors(CurDecomposition& c, const DevBuf<double>& dT, const DevBuf<double>& dS, Index l, Index k,
                        Index r) {
  const auto t = dT.download(), s = dS.download();
  c.tsig = Matrix(l, r);
  c.sr = Matrix(k, r);
  std::copy(t.begin(), t.begin() + l * r, c.tsig.data());
  std::copy(s.begin(), s.begin() + k * r, c.sr.data());
}

CurDecomposition primitive_cur(const EntryOracle& M, IndexSet I, IndexSet J, Index r, bool qr_nucleus) {
  // cur.cpp:137-162
  // r = 0 selects the adaptive rank (numerical_rank(G, 1e-10)); r < 0 is invalid
  if (I.size() < r || J.size() < r || r < 0)
    throw std::invalid_argument("primitive_cur: need |I|, |J| >= r >= 0 (0: adaptive rank)");
  if (I.bound() != M.rows() || J.bound() != M.cols()) throw std::invalid_argument("primitive_cur: index bounds");
  const DeviceMatrix& dA = M.device();
  const Index k = I.size(), l = J.size();
  DevBuf<int64_t> dI(to64(I)), dJ(to64(J));
  DeviceMatrix dU(l, k);
  if (qr_nucleus) {
    // cur.cpp:146-152: nucleus = G^+ by CompleteOrthogonalDecomposition
    // (threshold 1e-10), no rank-r truncation; rank() < r -> GeneratorRankFailure.
    // With r = 0 the COD rank is reported as r.
    DeviceMatrix dG(k, l);
    check(slra_gather_block(device_context(), dA.data(), dA.ld(), M.rows(), M.cols(), dI.get(), k, dJ.get(), l,
                            dG.data(), dG.ld()),
          "primitive_cur");
    int64_t rank = 0;
    check(slra_cod_pinv(device_context(), dG.data(), dG.ld(), k, l, 1e-10, dU.data(), l, &rank), "primitive_cur");
    M.count(static_cast<unsigned long long>(k * l));
    if (rank < std::max<Index>(r, 1)) throw GeneratorRankFailure("primitive_cur: generator rank below target");
    CurDecomposition c;
    c.row_set = std::move(I);
    c.col_set = std::move(J);
    c.nucleus = dU.download();
    c.r = r > 0 ? r : rank;
    c.qr_nucleus = true;
    return c;
  }
  const Index kl = std::min(k, l);
  DevBuf<double> dT(static_cast<size_t>(l * kl)), dS(static_cast<size_t>(k * kl));
  int64_t r_used = 0;
  check(slra_primitive_cur(device_context(), dA.data(), dA.ld(), M.rows(), M.cols(), dI.get(), k, dJ.get(), l, r,
                           dU.data(), l, dT.get(), dS.get(), &r_used),
        "primitive_cur");
  M.count(static_cast<unsigned long long>(k * l));  // the only entries read
  CurDecomposition c;
  c.row_set = std::move(I);
  c.col_set = std::move(J);
  c.nucleus = dU.download();
  c.r = r_used;
  set_factors(c, dT, dS, l, k, r_used);
  return c;
}

CurDecomposition primitive_cur(const Matrix& M, IndexSet I, IndexSet J, Index r, bool qr_nucleus) {
  DenseOracle o(M);
  return primitive_cur(o, std::move(I), std::move(J), r, qr_nucleus);
}

// cross_approx with the early stop (cur.cpp:235-249): after every horizontal
// half-sweep, primitive_cur probes the current generator and
// posterior_error_estimate (lra.cpp:88-127) samples q x s = 20 x 20 entries
// of M - C U R; the loop stops once the estimate is <= stop_tol. Host-driven
// half-sweeps over the device primitives (gather -> select_rows_spanning with
// its volume proxy); the sampled residual is a device GEMM + residual pass.
// The rng draws happen exactly where the reference draws them (only after a
// successful probe), so the caller's Rng stream matches.
static std::pair<CurDecomposition, CaTrace> cross_approx_stop(const EntryOracle& M, Index r, Index k, Index l,
                                                              IndexSet I, int loops, double h, double stop_tol,
                                                              Rng& rng) {
  slra_ctx cx = device_context();
  const DeviceMatrix& dA = M.device();
  const Index m = M.rows(), n = M.cols();
  DevBuf<int64_t> dI(to64(I)), dJ(static_cast<size_t>(l));
  DevBuf<double> ones(std::vector<double>(static_cast<size_t>(k), 1.0));
  DevBuf<double> RT(static_cast<size_t>(n * k)), Cm(static_cast<size_t>(m * l)), vol(1);
  CaTrace trace;
  IndexSet J;
  unsigned long long reads = 0;
  auto download_set = [](DevBuf<int64_t>& d, Index bound) {
    auto v = d.download();
    return IndexSet(std::vector<Index>(v.begin(), v.end()), bound);
  };
  for (int loop = 0; loop < loops; ++loop) {
    // J = select_rows_spanning(A(I,:)^T, l)
    check(slra_sketch_rows_shard(cx, dA.data(), dA.ld(), 0, m, n, dI.get(), ones.get(), 1, k, RT.get(), n, 1),
          "cross_approx");
    check(slra_select_rows_spanning(cx, RT.get(), n, n, k, l, h, dJ.get(), vol.get()), "cross_approx");
    J = download_set(dJ, n);
    CaStep sv;
    sv.horizontal = false;
    sv.rows.assign(I.begin(), I.end());
    sv.cols.assign(J.begin(), J.end());
    sv.volume_proxy = vol.download()[0];
    trace.steps.push_back(std::move(sv));
    // I = select_rows_spanning(A(:,J), k)
    check(slra_gather_cols(cx, dA.data(), dA.ld(), m, n, dJ.get(), l, Cm.get(), m), "cross_approx");
    check(slra_select_rows_spanning(cx, Cm.get(), m, m, l, k, h, dI.get(), vol.get()), "cross_approx");
    I = download_set(dI, m);
    reads += static_cast<unsigned long long>(k * n + m * l);
    CaStep st;
    st.horizontal = true;
    st.rows.assign(I.begin(), I.end());
    st.cols.assign(J.begin(), J.end());
    st.volume_proxy = vol.download()[0];
    try {
      const CurDecomposition probe = primitive_cur(M, I, J, r);
      // f.U = M(:,J) nucleus, f.V = M(I,:): sample q x s entries of M - U V
      const Index q = std::min<Index>(20, m), s = std::min<Index>(20, n);
      DevBuf<int64_t> dIs(to64(IndexSet(rng.distinct_indices(q, m), m)));
      DevBuf<int64_t> dJs(to64(IndexSet(rng.distinct_indices(s, n), n)));
      DeviceMatrix Xs(q, l), Rs(k, s), Ms(q, s), P(q, k);
      DeviceMatrix U = DeviceMatrix::upload(probe.nucleus);
      check(slra_gather_block(cx, dA.data(), dA.ld(), m, n, dIs.get(), q, dJ.get(), l, Xs.data(), q), "estimate");
      check(slra_gather_block(cx, dA.data(), dA.ld(), m, n, dI.get(), k, dJs.get(), s, Rs.data(), k), "estimate");
      check(slra_gather_block(cx, dA.data(), dA.ld(), m, n, dIs.get(), q, dJs.get(), s, Ms.data(), q), "estimate");
      check(slra_gemm(cx, 0, 0, q, k, l, 1.0, Xs.data(), q, U.data(), l, 0.0, P.data(), q), "estimate");
      DevBuf<double> out(2);
      check(slra_lowrank_residual(cx, Ms.data(), q, q, s, P.data(), q, Rs.data(), k, k, out.get()), "estimate");
      const double sumsq = out.download()[0];
      st.error_estimate = std::sqrt(static_cast<double>(m) * static_cast<double>(n) * sumsq /
                                    static_cast<double>(q * s));
      reads += static_cast<unsigned long long>(m * l + k * n + q * s);
    } catch (const GeneratorRankFailure&) {
      st.error_estimate.reset();
    }
    const bool stop = st.error_estimate && *st.error_estimate <= stop_tol;
    trace.steps.push_back(std::move(st));
    if (stop) break;
  }
  M.count(reads);
  auto c = primitive_cur(M, std::move(I), std::move(J), r);
  return {std::move(c), std::move(trace)};
}

std::pair<CurDecomposition, CaTrace> cross_approx(const EntryOracle& M, Index r, Index k, Index l,
                                                  IndexSet init_rows, int loops, double h,
                                                  std::optional<double> stop_tol, Rng& rng) {
  // cur.cpp:201-255
  const Index m = M.rows(), n = M.cols();
  if (k < r || l < r || r < 0) throw std::invalid_argument("cross_approx: need k, l >= r >= 1");
  if (loops < 1) throw std::invalid_argument("cross_approx: need loops >= 1");
  if (stop_tol && r < 1) throw std::invalid_argument("cross_approx: stop_tol needs a fixed r >= 1");
  IndexSet I = (init_rows.size() == k && init_rows.bound() == m) ? std::move(init_rows)
                                                                 : IndexSet(rng.distinct_indices(k, m), m);
  if (stop_tol) return cross_approx_stop(M, r, k, l, std::move(I), loops, h, *stop_tol, rng);
  const DeviceMatrix& dA = M.device();
  DevBuf<int64_t> dI0(to64(I)), dI(static_cast<size_t>(k)), dJ(static_cast<size_t>(l));
  DevBuf<int64_t> trows(static_cast<size_t>(2 * loops * k)), tcols(static_cast<size_t>(2 * loops * l));
  DevBuf<double> tvol(static_cast<size_t>(2 * loops));
  DeviceMatrix dU(l, k);
  const Index kl = std::min(k, l);
  DevBuf<double> dT(static_cast<size_t>(l * kl)), dS(static_cast<size_t>(k * kl));
  int64_t r_used = 0;
  check(slra_cross_approx(device_context(), dA.data(), dA.ld(), m, n, r, k, l, dI0.get(), loops, h, dI.get(),
                          dJ.get(), dU.data(), trows.get(), tcols.get(), tvol.get(), dT.get(), dS.get(), &r_used),
        "cross_approx");
  // algorithmic reads: per loop one k x n row strip and one m x l column
  // strip, then the k x l generator (the reference's DenseOracle count)
  M.count(static_cast<unsigned long long>(loops) * static_cast<unsigned long long>(k * n + m * l) +
          static_cast<unsigned long long>(k * l));
  auto vI = dI.download(), vJ = dJ.download(), tr = trows.download(), tc = tcols.download();
  auto tv = tvol.download();
  CaTrace trace;
  for (int s = 0; s < 2 * loops; ++s) {
    CaStep st;
    st.horizontal = (s % 2) == 1;
    st.rows.assign(tr.begin() + s * k, tr.begin() + (s + 1) * k);
    st.cols.assign(tc.begin() + s * l, tc.begin() + (s + 1) * l);
    st.volume_proxy = tv[static_cast<size_t>(s)];
    trace.steps.push_back(std::move(st));
  }
  CurDecomposition c;
  c.row_set = IndexSet(std::vector<Index>(vI.begin(), vI.end()), m);
  c.col_set = IndexSet(std::vector<Index>(vJ.begin(), vJ.end()), n);
  c.nucleus = dU.download();
  c.r = r_used;
  set_factors(c, dT, dS, l, k, r_used);
  return {std::move(c), std::move(trace)};
}

double cur_evaluate(const EntryOracle& M, const CurDecomposition& c, NormKind norm) {  // cur.cpp:80-82
  const DeviceMatrix& dA = M.device();
  DevBuf<int64_t> dI(to64(c.row_set)), dJ(to64(c.col_set));
  if (norm != NormKind::Frobenius) {
    // E = M - (C U) R formed on the device (cur.cpp:76-82), then its
    // spectral (SVD) or Chebyshev (max |e_ij|) norm
    slra_ctx cx = device_context();
    const Index m = M.rows(), n = M.cols(), k = c.row_set.size(), l = c.col_set.size();
    DeviceMatrix Cm(m, l), R(k, n), P(m, k), E(m, n), dU = DeviceMatrix::upload(c.nucleus);
    check(slra_gather_cols(cx, dA.data(), dA.ld(), m, n, dJ.get(), l, Cm.data(), Cm.ld()), "cur_evaluate");
    check(slra_gather_rows(cx, dA.data(), dA.ld(), m, n, dI.get(), k, R.data(), R.ld()), "cur_evaluate");
    check(slra_gemm(cx, 0, 0, m, k, l, 1.0, Cm.data(), Cm.ld(), dU.data(), dU.ld(), 0.0, P.data(), P.ld()),
          "cur_evaluate");
    check(slra_scale_rows_cols(cx, dA.data(), dA.ld(), m, n, nullptr, nullptr, E.data(), E.ld()), "cur_evaluate");
    check(slra_gemm(cx, 0, 0, m, n, k, -1.0, P.data(), P.ld(), R.data(), R.ld(), 1.0, E.data(), E.ld()),
          "cur_evaluate");
    M.count(static_cast<unsigned long long>(m * n + m * l + k * n));
    double v = 0.0;
    check(slra_matrix_norm(cx, E.data(), E.ld(), m, n, norm == NormKind::Spectral ? 0 : 2, &v), "cur_evaluate");
    return v;
  }
  if (c.r > 0 && c.tsig.cols() == c.r && c.sr.cols() == c.r) {
    // factored nucleus: the pass over M runs at inner dimension r
    DeviceMatrix dT = DeviceMatrix::upload(c.tsig), dS = DeviceMatrix::upload(c.sr);
    DevBuf<double> out(2);
    check(slra_cur_residual_factored(device_context(), dA.data(), dA.ld(), M.rows(), M.cols(), dI.get(),
                                     c.row_set.size(), dJ.get(), c.col_set.size(), dT.data(), dS.data(), c.r,
                                     out.get()),
          "cur_evaluate");
    return std::sqrt(out.download()[0]);
  }
  DeviceMatrix dU = DeviceMatrix::upload(c.nucleus);
  double rs = 0, ns = 0;
  check(slra_cur_residual(device_context(), dA.data(), dA.ld(), M.rows(), M.cols(), dI.get(), c.row_set.size(),
                          dJ.get(), c.col_set.size(), dU.data(), dU.ld(), &rs, &ns),
        "cur_evaluate");
  return std::sqrt(rs);
}

double cur_evaluate(const Matrix& M, const CurDecomposition& c, NormKind norm) {
  DenseOracle o(M);
  return cur_evaluate(o, c, norm);
}

Matrix cur_reconstruct(const Matrix& M, const CurDecomposition& c) {  // cur.cpp:76-78
  return matmul(matmul(select_cols(M, c.col_set), c.nucleus), select_rows(M, c.row_set));
}

// ---------------------------------------------------------------- oracle
const DeviceMatrix& DenseOracle::device() const {
  if (!dev_) dev_ = std::make_unique<DeviceMatrix>(DeviceMatrix::upload(*M_));
  return *dev_;
}

// ---------------------------------------------------------------- lra
void range_finder_device(const DeviceMatrix& M, const SketchPlan& plan, Index r, RangeVariant variant,
                         DeviceMatrix& U, DeviceMatrix& V, double* d_out) {
  DevBuf<int64_t> src(plan.src);
  DevBuf<double> coef(plan.coef);
  DevBuf<int32_t> q(plan.q);
  check(slra_range_finder(device_context(), M.data(), M.ld(), M.rows(), M.cols(), src.get(), coef.get(), q.get(),
                          plan.width, plan.tree, plan.count, r, variant == RangeVariant::TruncatedRankR ? 1 : 0,
                          U.data(), U.ld(), V.data(), V.ld(), d_out, nullptr),
        "range_finder");
}

LowRankFactors range_finder(const Matrix& M, const SketchOperator& H, Index r, RangeVariant variant) {
  // lra.cpp:14-39
  if (H.rows() != M.cols()) throw std::invalid_argument("range_finder: H rows != n");
  const Index l = H.cols();
  if (r < 1 || r > l) throw std::invalid_argument("range_finder: need 1 <= r <= l");
  const SketchPlan plan = compile_plan(H, Side::Right);
  DeviceMatrix dM = DeviceMatrix::upload(M);
  const Index uc = variant == RangeVariant::TruncatedRankR ? r : l;
  DeviceMatrix dU(M.rows(), uc), dV(uc, M.cols());
  range_finder_device(dM, plan, r, variant, dU, dV, nullptr);
  LowRankFactors f;
  f.U = dU.download();
  f.V = dV.download();
  f.target_rank = r;
  return f;
}

LowRankFactors lra_premult(const Matrix& M, const SketchOperator& F, const SketchOperator& H, Index r,
                           RangeVariant variant) {  // lra.cpp:41-52
  if (F.cols() != M.rows()) throw std::invalid_argument("lra_premult: F cols != m");
  if (H.rows() != M.cols()) throw std::invalid_argument("range_finder: H rows != n");
  const Index l = H.cols();
  if (r < 1 || r > l) throw std::invalid_argument("range_finder: need 1 <= r <= l");
  const SketchPlan ph = compile_plan(H, Side::Right), pf = compile_plan(F, Side::Left);
  DevBuf<int64_t> hs(ph.src), fs(pf.src);
  DevBuf<double> hc(ph.coef), fc(pf.coef);
  DevBuf<int32_t> hq(ph.q), fq(pf.q);
  DeviceMatrix dM = DeviceMatrix::upload(M);
  const Index uc = variant == RangeVariant::TruncatedRankR ? r : l;
  DeviceMatrix dU(M.rows(), uc), dV(uc, M.cols());
  check(slra_lra_premult(device_context(), dM.data(), dM.ld(), M.rows(), M.cols(), hs.get(), hc.get(), hq.get(),
                         ph.width, ph.tree, ph.count, fs.get(), fc.get(), fq.get(), pf.width, pf.tree, pf.count, r,
                         variant == RangeVariant::TruncatedRankR ? 1 : 0, dU.data(), dU.ld(), dV.data(), dV.ld(),
                         nullptr),
        "lra_premult");
  LowRankFactors f;
  f.U = dU.download();
  f.V = dV.download();
  f.target_rank = r;
  return f;
}

LowRankFactors two_stage_truncate(const LowRankFactors& f, Index r) {  // lra.cpp:54-63
  if (r < 1 || r > f.l()) throw std::invalid_argument("two_stage_truncate: need 1 <= r <= l");
  const Index m = f.U.rows(), n = f.V.cols();
  if (f.V.rows() != f.l()) throw std::invalid_argument("two_stage_truncate: U, V inner dimensions differ");
  DeviceMatrix dU = DeviceMatrix::upload(f.U), dV = DeviceMatrix::upload(f.V), dUo(m, r), dVo(r, n);
  check(slra_two_stage_truncate(device_context(), dU.data(), dU.ld(), m, f.l(), dV.data(), dV.ld(), n, r, dUo.data(),
                                dUo.ld(), dVo.data(), dVo.ld()),
        "two_stage_truncate");
  LowRankFactors out;
  out.U = dUo.download();
  out.V = dVo.download();
  out.target_rank = r;
  return out;
}

BatchedCaResult cross_approx_batched(const double* blocks, Index lda, Index block_stride, Index nblocks, Index m,
                                     Index n, Index r, Index k, Index l, const Index* init_rows, int loops, double h,
                                     Index* I_out, Index* J_out, double* nucleus_out) {
  if (nblocks < 0 || m < 1 || n < 1 || lda < m || block_stride < lda * n)
    throw std::invalid_argument("cross_approx_batched: bad block layout");
  if (k < 1 || l < 1 || k > m || l > n || (r > 0 && (r > k || r > l)))
    throw std::invalid_argument("cross_approx_batched: need r <= k <= m and r <= l <= n");
  BatchedCaResult out;
  out.status.resize(static_cast<size_t>(nblocks));
  out.r.resize(static_cast<size_t>(nblocks));
  out.resid_sq.resize(static_cast<size_t>(nblocks));
  out.norm_sq.resize(static_cast<size_t>(nblocks));
  std::vector<int32_t> st(static_cast<size_t>(nblocks));
  check(slra_cross_approx_batched_host(device_context(), blocks, lda, block_stride, nblocks, m, n, r, k, l,
                                       reinterpret_cast<const int64_t*>(init_rows), loops, h,
                                       reinterpret_cast<int64_t*>(I_out), reinterpret_cast<int64_t*>(J_out),
                                       nucleus_out, reinterpret_cast<int64_t*>(out.r.data()), st.data(),
                                       out.resid_sq.data(), out.norm_sq.data()),
        "cross_approx_batched");
  for (size_t b = 0; b < st.size(); ++b) out.status[b] = st[b];
  return out;
}

}  // namespace slra
