// HSS construction / products (/root/reference/proj/src/hss.cpp) over the
// C-ABI. The matrix stays in HBM; blocks are windows of it (pointer + ld),
// never copies. Svd strategy: one C-ABI call (slra_hss_build_svd). CurCa
// strategy: the reference's per-block binary search (hss.cpp:98-141) is
// host-driven because every step draws from the caller's Rng and branches on
// the previous estimate; each step is a device cross-approximation plus a
// device-sampled error estimate.
#include "slra/hss.hpp"

#include <cmath>
#include <functional>
#include <sstream>
#include <stdexcept>

#include "slra/cur.hpp"
#include "slra/errors.hpp"

namespace slra {

namespace {

// hss.cpp:16-31: a window of another oracle (device view, shared counter)
class BlockOracle final : public EntryOracle {
 public:
  BlockOracle(const EntryOracle& base, Index row0, Index col0, Index rows, Index cols)
      : base_(base),
        view_(DeviceMatrix::view(base.device().data() + row0 + col0 * base.device().ld(), rows, cols,
                                 base.device().ld())) {}
  Index rows() const override { return view_.rows(); }
  Index cols() const override { return view_.cols(); }
  const DeviceMatrix& device() const override { return view_; }
  void count(unsigned long long n) const override { base_.count(n); }

 private:
  const EntryOracle& base_;
  DeviceMatrix view_;
};

std::vector<int64_t> to64(const std::vector<Index>& v) { return std::vector<int64_t>(v.begin(), v.end()); }

// Reference block order (hss.cpp:151-160): preorder over internal nodes,
// upper then lower block. Calls f(level, node).
void preorder(int L, const std::function<void(int, Index)>& f) {
  std::function<void(int, Index)> visit = [&](int l, Index t) {
    f(l, t);
    if (l + 1 < L) {
      visit(l + 1, 2 * t);
      visit(l + 1, 2 * t + 1);
    }
  };
  visit(0, 0);
}

Index level_base(int l) { return (Index(2) << l) - 2; }

void validate(Index n, int L, Index r) {
  // hss.cpp:167-172
  if (L < 1) throw std::invalid_argument("build_hss: depth >= 1");
  const Index blocks = Index(1) << L;
  if (n % blocks != 0) throw std::invalid_argument("build_hss: n not divisible by 2^L");
  if (n / blocks < r) throw std::invalid_argument("build_hss: leaf size below rank");
}

// posterior_error_estimate's Frobenius estimate (lra.cpp:88-115) of B - F R
// on a q x s sample drawn from rng (rows first, then columns): the sampled
// residual entries are one gather + one low-rank residual pass on the device.
// F (rows x rho, ld rows) and R (rho x cols, ld rho) are device buffers;
// rho = 0 samples B itself (hss.cpp:33-44 zero factors).
double sampled_frobenius(const BlockOracle& B, const double* F, const double* R, Index rho, Rng& rng) {
  slra_ctx cx = device_context();
  const Index m = B.rows(), n = B.cols();
  const Index q = std::min<Index>(20, m), s = std::min<Index>(20, n);
  if (q * s < 2) throw std::invalid_argument("posterior_error_estimate: bad sample sizes");  // lra.cpp:94-95
  DevBuf<int64_t> I(to64(rng.distinct_indices(q, m))), J(to64(rng.distinct_indices(s, n)));
  const DeviceMatrix& d = B.device();
  DevBuf<double> Ms(static_cast<size_t>(q * s)), Fs(static_cast<size_t>(q * (rho > 0 ? rho : 1))),
      Rs(static_cast<size_t>((rho > 0 ? rho : 1) * s)), out(2);
  check(slra_gather_block(cx, d.data(), d.ld(), m, n, I.get(), q, J.get(), s, Ms.get(), q), "hss estimate");
  if (rho > 0) {
    check(slra_gather_rows(cx, F, m, m, rho, I.get(), q, Fs.get(), q), "hss estimate");
    check(slra_gather_cols(cx, R, rho, rho, n, J.get(), s, Rs.get(), rho), "hss estimate");
  }
  check(slra_lowrank_residual(cx, Ms.get(), q, q, s, rho > 0 ? Fs.get() : nullptr, q, rho > 0 ? Rs.get() : nullptr,
                              rho > 0 ? rho : 1, rho, out.get()),
        "hss estimate");
  B.count(static_cast<unsigned long long>(q * s));
  const double sumsq = out.download()[0];
  return std::sqrt(static_cast<double>(m) * static_cast<double>(n) * sumsq / static_cast<double>(q * s));
}

struct CaCandidate {
  std::vector<Index> I, J;
  Matrix nucleus;
  Index rho = 0;
};

// hss.cpp:46-56 ca_factors: C-A at rank rho (k = l = rho, 2 loops, h 1.1),
// F = B(:, J) nucleus, V = B(I, :), then the sampled error estimate.
std::pair<CaCandidate, double> ca_factors(const BlockOracle& B, Index rho, Rng& rng) {
  slra_ctx cx = device_context();
  auto [c, trace] = cross_approx(B, rho, rho, rho, IndexSet(), 2, 1.1, std::nullopt, rng);
  (void)trace;
  const Index m = B.rows(), n = B.cols();
  const DeviceMatrix& d = B.device();
  DevBuf<int64_t> dI(std::vector<int64_t>(c.row_set.begin(), c.row_set.end()));
  DevBuf<int64_t> dJ(std::vector<int64_t>(c.col_set.begin(), c.col_set.end()));
  DevBuf<double> Cm(static_cast<size_t>(m * rho)), F(static_cast<size_t>(m * rho)), R(static_cast<size_t>(rho * n));
  DeviceMatrix U = DeviceMatrix::upload(c.nucleus);  // l x k = rho x rho
  check(slra_gather_cols(cx, d.data(), d.ld(), m, n, dJ.get(), rho, Cm.get(), m), "ca_factors");
  check(slra_gemm(cx, 0, 0, m, rho, rho, 1.0, Cm.get(), m, U.data(), U.ld(), 0.0, F.get(), m), "ca_factors");
  check(slra_gather_rows(cx, d.data(), d.ld(), m, n, dI.get(), rho, R.get(), rho), "ca_factors");
  B.count(static_cast<unsigned long long>(m * rho + rho * n));  // cols_of + rows_of
  CaCandidate cand;
  cand.I.assign(c.row_set.begin(), c.row_set.end());
  cand.J.assign(c.col_set.begin(), c.col_set.end());
  cand.nucleus = std::move(c.nucleus);
  cand.rho = rho;
  const double err = sampled_frobenius(B, F.get(), R.get(), rho, rng);
  return {std::move(cand), err};
}

// Writes a candidate's generators into the packed level arrays:
// F_l(row0 + i, :) = (B(:, J) nucleus)(i, :), HT_l(col0 + j, :) = B(I, j)^T.
void emit_candidate(const BlockOracle& B, const CaCandidate& c, double* Fl, double* HTl, Index n, Index row0,
                    Index col0) {
  slra_ctx cx = device_context();
  const Index m = B.rows(), nc = B.cols(), rho = c.rho;
  const DeviceMatrix& d = B.device();
  DevBuf<int64_t> dI(to64(c.I)), dJ(to64(c.J));
  DevBuf<double> Cm(static_cast<size_t>(m * rho)), ones(std::vector<double>(static_cast<size_t>(rho), 1.0));
  DeviceMatrix U = DeviceMatrix::upload(c.nucleus);
  check(slra_gather_cols(cx, d.data(), d.ld(), m, nc, dJ.get(), rho, Cm.get(), m), "hss emit");
  check(slra_gemm(cx, 0, 0, m, rho, rho, 1.0, Cm.get(), m, U.data(), U.ld(), 0.0, Fl + row0, n), "hss emit");
  check(slra_sketch_rows_shard(cx, d.data(), d.ld(), 0, m, nc, dI.get(), ones.get(), 1, rho, HTl + col0, n, 1),
        "hss emit");
}

// hss.cpp:98-141 (superfast path): returns the block's rank and overflow.
std::pair<Index, bool> approx_block_ca(const EntryOracle& M, Index row0, Index col0, Index rows, Index cols,
                                       Index r, double tol, Rng& rng, double* Fl, double* HTl, Index n) {
  BlockOracle B(M, row0, col0, rows, cols);
  const double scale = sampled_frobenius(B, nullptr, nullptr, 0, rng);
  if (scale <= 0) return {0, false};
  const Index cap = std::min(r, std::min(rows, cols));
  CaCandidate accepted, fallback;
  double fallback_err = -1;
  bool have_accepted = false;
  Index lo = 1, hi = cap;
  while (lo <= hi) {
    const Index mid = (lo + hi) / 2;
    try {
      auto [c, err] = ca_factors(B, mid, rng);
      if (err <= tol * scale) {
        accepted = std::move(c);
        have_accepted = true;
        hi = mid - 1;
      } else {
        if (fallback_err < 0 || err < fallback_err) {
          fallback = std::move(c);
          fallback_err = err;
        }
        lo = mid + 1;
      }
    } catch (const GeneratorRankFailure&) {
      hi = mid - 1;
    } catch (const SelectionFailure&) {
      hi = mid - 1;
    }
  }
  if (have_accepted) {
    emit_candidate(B, accepted, Fl, HTl, n, row0, col0);
    return {accepted.rho, false};
  }
  if (fallback_err >= 0) {
    emit_candidate(B, fallback, Fl, HTl, n, row0, col0);
    return {fallback.rho, true};
  }
  return {0, true};
}

HssDevice alloc_device(Index n, int L, Index r) {
  HssDevice h;
  h.n = n;
  h.depth = L;
  h.leaf = n >> L;
  h.r = r;
  const size_t fr = static_cast<size_t>(L) * static_cast<size_t>(n) * static_cast<size_t>(r > 0 ? r : 1);
  h.D = DevBuf<double>(static_cast<size_t>(n * h.leaf));
  h.F = DevBuf<double>(fr);
  h.HT = DevBuf<double>(fr);
  const size_t nb = static_cast<size_t>(level_base(L));
  h.rank = DevBuf<int64_t>(nb);
  h.h_rank.assign(nb, 0);
  h.h_overflow.assign(nb, 0);
  return h;
}

void block_geometry(Index n, int l, Index t, int side, Index& row0, Index& col0, Index& half) {
  const Index size = n >> l;
  half = size / 2;
  row0 = t * size + (side ? half : 0);
  col0 = t * size + (side ? 0 : half);
}

}  // namespace

HssDevice build_hss_device(const EntryOracle& M, int L, Index r, double tol, HssStrategy strategy, Rng& rng) {
  const Index n = M.rows();
  if (M.cols() != n) throw std::invalid_argument("build_hss: matrix must be square");
  validate(n, L, r);
  slra_ctx cx = device_context();
  const DeviceMatrix& d = M.device();
  HssDevice h = alloc_device(n, L, r);
  if (strategy == HssStrategy::Svd) {
    check(slra_hss_build_svd(cx, d.data(), d.ld(), n, L, r, tol, h.D.get(), h.F.get(), h.HT.get(), h.h_rank.data(),
                             h.h_overflow.data()),
          "build_hss");
    h.rank.upload(h.h_rank);
    M.count(static_cast<unsigned long long>(n * n));  // B.dense() of every block and leaf
    return h;
  }
  // CurCa: the reference's recursion order (hss.cpp:143-161) fixes the Rng stream
  check(slra_hss_leaves(cx, d.data(), d.ld(), n, L, h.D.get()), "build_hss");
  // generator columns >= a block's rank are never read (every kernel and the
  // download stop at rank[g]), so the packed arrays need no clearing
  preorder(L, [&](int l, Index t) {
    for (int side = 0; side < 2; ++side) {
      Index row0, col0, half;
      block_geometry(n, l, t, side, row0, col0, half);
      const size_t off = static_cast<size_t>(l) * static_cast<size_t>(n) * static_cast<size_t>(r);
      auto [rho, over] =
          approx_block_ca(M, row0, col0, half, half, r, tol, rng, h.F.get() + off, h.HT.get() + off, n);
      const size_t g = static_cast<size_t>(level_base(l) + 2 * t + side);
      h.h_rank[g] = rho;
      h.h_overflow[g] = over ? 1 : 0;
    }
  });
  M.count(static_cast<unsigned long long>(n * h.leaf));  // the dense leaves
  h.rank.upload(h.h_rank);
  return h;
}

HssMatrix hss_download(const HssDevice& h) {
  const Index n = h.n, r = h.r;
  HssMatrix out;
  out.n = n;
  out.depth = h.depth;
  out.leaf = h.leaf;
  out.r = r;
  const std::vector<double> D = h.D.download();
  for (Index t = 0; t < (Index(1) << h.depth); ++t) {
    HssLeaf leaf;
    leaf.row0 = leaf.col0 = t * h.leaf;
    leaf.D = Matrix(h.leaf, h.leaf);
    for (Index j = 0; j < h.leaf; ++j)
      for (Index i = 0; i < h.leaf; ++i) leaf.D(i, j) = D[static_cast<size_t>(t * h.leaf + i + j * n)];
    out.diag.push_back(std::move(leaf));
  }
  std::vector<double> F, HT;
  if (r > 0) {
    F = h.F.download();
    HT = h.HT.download();
  }
  preorder(h.depth, [&](int l, Index t) {
    for (int side = 0; side < 2; ++side) {
      HssBlock b;
      Index half;
      block_geometry(n, l, t, side, b.row0, b.col0, half);
      b.rows = b.cols = half;
      const size_t g = static_cast<size_t>(level_base(l) + 2 * t + side);
      const Index rho = h.h_rank[g];
      b.rank_overflow = h.h_overflow[g] != 0;
      b.F = Matrix(half, rho);
      b.H = Matrix(rho, half);
      const size_t off = static_cast<size_t>(l) * static_cast<size_t>(n) * static_cast<size_t>(r);
      for (Index a = 0; a < rho; ++a)
        for (Index i = 0; i < half; ++i) {
          b.F(i, a) = F[off + static_cast<size_t>(b.row0 + i + a * n)];
          b.H(a, i) = HT[off + static_cast<size_t>(b.col0 + i + a * n)];
        }
      out.any_overflow = out.any_overflow || b.rank_overflow;
      out.off.push_back(std::move(b));
    }
  });
  return out;
}

HssDevice hss_upload(const HssMatrix& H) {
  const Index n = H.n, r = H.r;
  const int L = H.depth;
  validate(n, L, r);
  if (H.leaf != (n >> L) || static_cast<Index>(H.diag.size()) != (Index(1) << L) ||
      static_cast<Index>(H.off.size()) != level_base(L))
    throw std::invalid_argument("hss: not a depth-L binary partition");
  HssDevice h = alloc_device(n, L, r);
  std::vector<double> D(static_cast<size_t>(n * h.leaf), 0.0);
  for (Index t = 0; t < static_cast<Index>(H.diag.size()); ++t) {
    const HssLeaf& leaf = H.diag[static_cast<size_t>(t)];
    if (leaf.row0 != t * h.leaf || leaf.col0 != t * h.leaf || leaf.D.rows() != h.leaf || leaf.D.cols() != h.leaf)
      throw std::invalid_argument("hss: leaf geometry");
    for (Index j = 0; j < h.leaf; ++j)
      for (Index i = 0; i < h.leaf; ++i) D[static_cast<size_t>(t * h.leaf + i + j * n)] = leaf.D(i, j);
  }
  const size_t fr = static_cast<size_t>(L) * static_cast<size_t>(n) * static_cast<size_t>(r > 0 ? r : 1);
  std::vector<double> F(fr, 0.0), HT(fr, 0.0);
  size_t k = 0;
  preorder(L, [&](int l, Index t) {
    for (int side = 0; side < 2; ++side, ++k) {
      const HssBlock& b = H.off[k];
      Index row0, col0, half;
      block_geometry(n, l, t, side, row0, col0, half);
      const Index rho = b.F.cols();
      if (b.row0 != row0 || b.col0 != col0 || b.rows != half || b.cols != half || rho > r || b.F.rows() != half ||
          b.H.rows() != rho || b.H.cols() != half)
        throw std::invalid_argument("hss: block geometry");
      const size_t g = static_cast<size_t>(level_base(l) + 2 * t + side);
      h.h_rank[g] = rho;
      h.h_overflow[g] = b.rank_overflow ? 1 : 0;
      const size_t off = static_cast<size_t>(l) * static_cast<size_t>(n) * static_cast<size_t>(r);
      for (Index a = 0; a < rho; ++a)
        for (Index i = 0; i < half; ++i) {
          F[off + static_cast<size_t>(row0 + i + a * n)] = b.F(i, a);
          HT[off + static_cast<size_t>(col0 + i + a * n)] = b.H(a, i);
        }
    }
  });
  h.D.upload(D);
  h.F.upload(F);
  h.HT.upload(HT);
  h.rank.upload(h.h_rank);
  return h;
}

HssMatrix build_hss(const EntryOracle& M, int L, Index r, double tol, HssStrategy strategy, Rng& rng) {
  return hss_download(build_hss_device(M, L, r, tol, strategy, rng));
}

HssMatrix build_hss(const Matrix& M, int L, Index r, double tol, HssStrategy strategy, Rng& rng) {
  DenseOracle o(M);
  return build_hss(o, L, r, tol, strategy, rng);
}

void hss_matvec_device(const HssDevice& h, const double* d_x, double* d_y) {
  check(slra_hss_matvec(device_context(), h.n, h.depth, h.r, h.D.get(), h.F.get(), h.HT.get(), h.rank.get(), d_x,
                        d_y),
        "hss_matvec");
}

Vector hss_matvec(const HssMatrix& H, const Vector& x) {  // hss.cpp:193-212
  if (static_cast<Index>(x.size()) != H.n) throw std::invalid_argument("hss_matvec: length mismatch");
  const HssDevice h = hss_upload(H);
  DevBuf<double> dx(x), dy(x.size());
  hss_matvec_device(h, dx.get(), dy.get());
  return dy.download();
}

Matrix hss_reconstruct(const HssMatrix& H) {  // hss.cpp:214-221
  const HssDevice h = hss_upload(H);
  DeviceMatrix R(H.n, H.n);
  check(slra_hss_reconstruct(device_context(), h.n, h.depth, h.r, h.D.get(), h.F.get(), h.HT.get(), h.rank.get(),
                             nullptr, 0, R.data(), R.ld()),
        "hss_reconstruct");
  return R.download();
}

double hss_error(const HssMatrix& H, const Matrix& M, NormKind norm) {  // hss.cpp:223-225
  if (M.rows() != H.n || M.cols() != H.n) throw std::invalid_argument("hss_error: shape mismatch");
  const HssDevice h = hss_upload(H);
  DeviceMatrix dM = DeviceMatrix::upload(M), E(H.n, H.n);
  check(slra_hss_reconstruct(device_context(), h.n, h.depth, h.r, h.D.get(), h.F.get(), h.HT.get(), h.rank.get(),
                             dM.data(), dM.ld(), E.data(), E.ld()),
        "hss_error");
  double v = 0.0;
  const int kind = norm == NormKind::Spectral ? 0 : norm == NormKind::Frobenius ? 1 : 2;
  check(slra_matrix_norm(device_context(), E.data(), E.ld(), H.n, H.n, kind, &v), "hss_error");
  return v;
}

// hss.cpp:227-291: the reference's text format, field for field.
std::string HssMatrix::serialize() const {
  std::ostringstream out;
  out.precision(17);
  out << "hss " << n << " " << depth << " " << leaf << " " << r << " " << (any_overflow ? 1 : 0) << " "
      << diag.size() << " " << off.size() << "\n";
  auto dump = [&out](const Matrix& M) {
    out << M.rows() << " " << M.cols();
    for (Index j = 0; j < M.cols(); ++j)
      for (Index i = 0; i < M.rows(); ++i) out << " " << M(i, j);
    out << "\n";
  };
  for (const HssLeaf& l : diag) {
    out << "leaf " << l.row0 << " " << l.col0 << "\n";
    dump(l.D);
  }
  for (const HssBlock& b : off) {
    out << "block " << b.row0 << " " << b.col0 << " " << b.rows << " " << b.cols << " " << (b.rank_overflow ? 1 : 0)
        << "\n";
    dump(b.F);
    dump(b.H);
  }
  return out.str();
}

HssMatrix HssMatrix::deserialize(const std::string& text) {
  std::istringstream in(text);
  std::string tag;
  HssMatrix h;
  int overflow = 0;
  size_t nleaf = 0, noff = 0;
  if (!(in >> tag >> h.n >> h.depth >> h.leaf >> h.r >> overflow >> nleaf >> noff) || tag != "hss")
    throw std::runtime_error("HssMatrix: bad header");
  h.any_overflow = overflow != 0;
  auto load = [&in](Matrix& M) {
    Index rows = 0, cols = 0;
    if (!(in >> rows >> cols) || rows < 0 || cols < 0) throw std::runtime_error("HssMatrix: bad matrix");
    M = Matrix(rows, cols);
    for (Index j = 0; j < cols; ++j)
      for (Index i = 0; i < rows; ++i)
        if (!(in >> M(i, j))) throw std::runtime_error("HssMatrix: bad matrix");
  };
  for (size_t t = 0; t < nleaf; ++t) {
    HssLeaf l;
    if (!(in >> tag >> l.row0 >> l.col0) || tag != "leaf") throw std::runtime_error("HssMatrix: bad leaf");
    load(l.D);
    h.diag.push_back(std::move(l));
  }
  for (size_t t = 0; t < noff; ++t) {
    HssBlock b;
    int ov = 0;
    if (!(in >> tag >> b.row0 >> b.col0 >> b.rows >> b.cols >> ov) || tag != "block")
      throw std::runtime_error("HssMatrix: bad block");
    b.rank_overflow = ov != 0;
    load(b.F);
    load(b.H);
    h.off.push_back(std::move(b));
  }
  return h;
}

}  // namespace slra
