// TEST INFRASTRUCTURE ONLY: Python binding of the CPU oracle for tests/ and
// bench.py's CPU legs. Not part of the product.
#include <pybind11/complex.h>
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <chrono>

#include "slra_oracle.hpp"

namespace py = pybind11;
using namespace slra_oracle;

using FArray = py::array_t<double, py::array::f_style | py::array::forcecast>;

static Matrix from_np(const FArray& a) {
  if (a.ndim() == 1) {
    Matrix M(a.shape(0), 1);
    std::copy(a.data(), a.data() + a.shape(0), M.v.begin());
    return M;
  }
  if (a.ndim() != 2) throw std::invalid_argument("expected a 1-D or 2-D array");
  Matrix M(a.shape(0), a.shape(1));
  std::copy(a.data(), a.data() + M.size(), M.v.begin());
  return M;
}
static FArray to_np(const Matrix& M) {
  FArray a({M.rows(), M.cols()});
  std::copy(M.v.begin(), M.v.end(), a.mutable_data());
  return a;
}
static py::array_t<double> vec_np(const Vector& v) {
  py::array_t<double> a(static_cast<py::ssize_t>(v.size()));
  std::copy(v.begin(), v.end(), a.mutable_data());
  return a;
}
static Vector np_vec(const FArray& a) { return Vector(a.data(), a.data() + a.size()); }
struct PyOp { OpPtr p; };
static IndexSet mkset(const std::vector<Index>& v, Index bound) { return IndexSet(v, bound); }


static py::dict hss_dict(const HssMatrix& h) {
  py::dict d;
  d["n"] = h.n;
  d["depth"] = h.depth;
  d["leaf"] = h.leaf;
  d["r"] = h.r;
  d["any_overflow"] = h.any_overflow;
  py::list diag, off;
  for (const HssLeaf& l : h.diag) diag.append(py::make_tuple(l.row0, l.col0, to_np(l.D)));
  for (const HssBlock& b : h.off) {
    py::dict e;
    e["row0"] = b.row0;
    e["col0"] = b.col0;
    e["rows"] = b.rows;
    e["cols"] = b.cols;
    e["F"] = to_np(b.F);
    e["H"] = to_np(b.H);
    e["rank_overflow"] = b.rank_overflow;
    off.append(e);
  }
  d["diag"] = diag;
  d["off"] = off;
  return d;
}

static HssMatrix hss_from(const py::dict& d) {
  HssMatrix h;
  h.n = d["n"].cast<Index>();
  h.depth = d["depth"].cast<int>();
  h.leaf = d["leaf"].cast<Index>();
  h.r = d["r"].cast<Index>();
  h.any_overflow = d["any_overflow"].cast<bool>();
  for (auto t : d["diag"].cast<py::list>()) {
    auto tp = t.cast<py::tuple>();
    HssLeaf l;
    l.row0 = tp[0].cast<Index>();
    l.col0 = tp[1].cast<Index>();
    l.D = from_np(tp[2].cast<FArray>());
    h.diag.push_back(std::move(l));
  }
  for (auto e : d["off"].cast<py::list>()) {
    auto b = e.cast<py::dict>();
    HssBlock k;
    k.row0 = b["row0"].cast<Index>();
    k.col0 = b["col0"].cast<Index>();
    k.rows = b["rows"].cast<Index>();
    k.cols = b["cols"].cast<Index>();
    k.F = from_np(b["F"].cast<FArray>());
    k.H = from_np(b["H"].cast<FArray>());
    if (k.F.cols() == 0) k.F = Matrix(k.rows, 0);
    if (k.H.rows() == 0) k.H = Matrix(0, k.cols);
    k.rank_overflow = b["rank_overflow"].cast<bool>();
    h.off.push_back(std::move(k));
  }
  return h;
}

static py::dict cur_dict(const CurDecomposition& c) {
  py::dict d;
  d["I"] = c.row_set.indices();
  d["J"] = c.col_set.indices();
  d["nucleus"] = to_np(c.nucleus);
  d["r"] = c.r;
  return d;
}

PYBIND11_MODULE(_oracle, m) {
  m.doc() = "CPU oracle (restatement of the reference slra hot path) -- test infrastructure only";
  auto base = py::register_local_exception<std::runtime_error>(m, "OracleRuntimeError");
  py::register_local_exception<RangeFailure>(m, "RangeFailure", base.ptr());
  py::register_local_exception<SketchRankFailure>(m, "SketchRankFailure", base.ptr());
  py::register_local_exception<PremultRankFailure>(m, "PremultRankFailure", base.ptr());
  py::register_local_exception<SelectionFailure>(m, "SelectionFailure", base.ptr());
  py::register_local_exception<GeneratorRankFailure>(m, "GeneratorRankFailure", base.ptr());
  py::register_local_exception<EmptySample>(m, "EmptySample", base.ptr());

  py::class_<Rng>(m, "Rng", py::module_local())
      .def(py::init<std::uint64_t>())
      .def("next_u64", &Rng::next_u64)
      .def("uniform", &Rng::uniform)
      .def("gaussian", &Rng::gaussian)
      .def("uniform_index", &Rng::uniform_index)
      .def("sign", &Rng::sign)
      .def("permutation", &Rng::permutation)
      .def("distinct_indices", &Rng::distinct_indices)
      .def("gaussian_matrix", [](Rng& r, Index a, Index b) { return to_np(r.gaussian_matrix(a, b)); })
      .def("gaussian_vector", [](Rng& r, Index n) { return vec_np(r.gaussian_vector(n)); })
      .def("child", &Rng::child)
      .def_static("derive_seed", &Rng::derive_seed);

  // ---- linalg
  m.def("matmul", [](const FArray& A, const FArray& B) { return to_np(matmul(from_np(A), from_np(B))); });
  m.def("thin_qr", [](const FArray& A) {
    auto [Q, R] = thin_qr(from_np(A));
    return py::make_tuple(to_np(Q), to_np(R));
  });
  m.def("svd", [](const FArray& A) {
    Svd f = svd(from_np(A));
    return py::make_tuple(to_np(f.S), vec_np(f.sigma), to_np(f.T));
  });
  m.def("pseudo_inverse", [](const FArray& A, double tol) { return to_np(pseudo_inverse(from_np(A), tol)); },
        py::arg("A"), py::arg("rank_tol") = 1e-10);
  m.def("numerical_rank", [](const FArray& A, double tol, bool relative) {
    return numerical_rank(from_np(A), tol, relative ? RankMode::Relative : RankMode::Absolute);
  }, py::arg("A"), py::arg("tol"), py::arg("relative") = false);
  m.def("frobenius_norm", [](const FArray& A) { return frobenius_norm(from_np(A)); });
  m.def("spectral_norm", [](const FArray& A) { return spectral_norm(from_np(A)); });
  m.def("determinant_abs", [](const FArray& A) { return determinant_abs(from_np(A)); });
  m.def("colpiv_qr", [](const FArray& A, double threshold) {
    ColPivQR q(from_np(A));
    q.threshold = threshold;
    py::dict d;
    d["perm"] = q.perm;
    d["rank"] = q.rank();
    d["nonzero_pivots"] = q.nonzero_pivots;
    d["qr"] = to_np(q.qr);
    return d;
  }, py::arg("A"), py::arg("threshold") = -1.0);
  m.def("colpiv_solve", [](const FArray& A, const FArray& B, double threshold) {
    ColPivQR q(from_np(A));
    q.threshold = threshold;
    return to_np(q.solve(from_np(B)));
  }, py::arg("A"), py::arg("B"), py::arg("threshold") = -1.0);

  // ---- cur
  m.def("t_factor", &t_factor);
  m.def("maxvol_rows", [](const FArray& A, double h, Index max_swaps) {
    return maxvol_rows(from_np(A), h, max_swaps).indices();
  }, py::arg("A"), py::arg("h") = 1.1, py::arg("max_swaps") = 0);
  m.def("select_rows_spanning", [](const FArray& A, Index count, double h) {
    return select_rows_spanning(from_np(A), count, h).indices();
  }, py::arg("A"), py::arg("count"), py::arg("h") = 1.1);
  m.def("primitive_cur", [](const FArray& A, const std::vector<Index>& I, const std::vector<Index>& J, Index r,
                            bool qr_nucleus) {
    Matrix M = from_np(A);
    DenseOracle o(M);
    py::dict d = cur_dict(primitive_cur(o, mkset(I, M.rows()), mkset(J, M.cols()), r, qr_nucleus));
    d["accesses"] = o.accesses();
    return d;
  }, py::arg("A"), py::arg("I"), py::arg("J"), py::arg("r"), py::arg("qr_nucleus") = false);
  m.def("cod_pseudo_inverse", [](const FArray& G, double threshold) {
    Index rank = 0;
    Matrix P = cod_pseudo_inverse(from_np(G), threshold, &rank);
    return py::make_tuple(to_np(P), rank);
  }, py::arg("G"), py::arg("threshold") = 1e-10);
  m.def("cross_approx", [](const FArray& A, Index r, Index k, Index l, const std::vector<Index>& init_rows,
                           int loops, double h, std::optional<double> stop_tol, Rng& rng) {
    Matrix M = from_np(A);
    DenseOracle o(M);
    IndexSet init = init_rows.empty() ? IndexSet() : mkset(init_rows, M.rows());
    auto [c, trace] = cross_approx(o, r, k, l, std::move(init), loops, h, stop_tol, rng);
    py::dict d = cur_dict(c);
    py::list steps;
    for (auto& s : trace.steps) {
      py::dict sd;
      sd["horizontal"] = s.horizontal;
      sd["rows"] = s.rows;
      sd["cols"] = s.cols;
      sd["volume_proxy"] = s.volume_proxy;
      sd["error_estimate"] = s.error_estimate;
      steps.append(sd);
    }
    d["trace"] = steps;
    d["accesses"] = o.accesses();
    return d;
  }, py::arg("A"), py::arg("r"), py::arg("k"), py::arg("l"), py::arg("init_rows"), py::arg("loops"),
     py::arg("h"), py::arg("stop_tol"), py::arg("rng"));
  // The config-5 batch through the restated reference path, block by block
  // (hss.cpp:47-55 pattern: cross_approx -> adaptive-rank primitive_cur ->
  // cur_evaluate), blocks spread over `threads` OpenMP threads (the reference
  // itself is single-threaded; threads = 1 is its literal execution). Block b
  // is the m x n column-major matrix at A + b*stride (ld = lda); host memory.
  m.def("cross_approx_blocks", [](uintptr_t Aptr, Index nb, Index mm, Index n, Index lda, Index stride,
                                  const py::array_t<Index, py::array::c_style | py::array::forcecast>& inits, Index k,
                                  Index l, int loops, double h, int threads) {
    const double* A = reinterpret_cast<const double*>(Aptr);
    py::array_t<Index> I({nb, k}), J({nb, l}), rr(nb);
    py::array_t<double> rs(nb), ns(nb);
    py::array_t<int> st(nb);
    const Index* ini = inits.data();
    Index* Ip = I.mutable_data();
    Index* Jp = J.mutable_data();
    Index* rp = rr.mutable_data();
    double* rsp = rs.mutable_data();
    double* nsp = ns.mutable_data();
    int* stp = st.mutable_data();
    {
      py::gil_scoped_release nogil;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
      for (Index b = 0; b < nb; ++b) {
        Matrix M(mm, n);
        for (Index j = 0; j < n; ++j)
          for (Index i = 0; i < mm; ++i) M(i, j) = A[b * stride + i + j * lda];
        double nrm = 0;
        for (double v : M.v) nrm += v * v;
        nsp[b] = nrm;
        try {
          DenseOracle o(M);
          Rng rng(0);
          std::vector<Index> init(ini + b * k, ini + (b + 1) * k);
          auto res = cross_approx(o, 1, k, l, IndexSet(init, mm), loops, h, std::nullopt, rng);
          const auto& Is = res.first.row_set.indices();
          const auto& Js = res.first.col_set.indices();
          Matrix G(k, l);
          for (Index j = 0; j < l; ++j)
            for (Index i = 0; i < k; ++i) G(i, j) = M(Is[static_cast<size_t>(i)], Js[static_cast<size_t>(j)]);
          const Index rk = numerical_rank(G, 1e-10, RankMode::Relative);
          CurDecomposition c = primitive_cur(M, res.first.row_set, res.first.col_set, rk);
          const double e = cur_evaluate(M, c, NormKind::Frobenius);
          for (Index i = 0; i < k; ++i) Ip[b * k + i] = Is[static_cast<size_t>(i)];
          for (Index j = 0; j < l; ++j) Jp[b * l + j] = Js[static_cast<size_t>(j)];
          rp[b] = rk;
          rsp[b] = e * e;
          stp[b] = 0;
        } catch (const std::exception&) {
          rp[b] = 0;
          rsp[b] = nrm;
          stp[b] = 1;
        }
      }
    }
    py::dict d;
    d["I"] = I;
    d["J"] = J;
    d["r"] = rr;
    d["resid_sq"] = rs;
    d["norm_sq"] = ns;
    d["status"] = st;
    return d;
  }, py::arg("A"), py::arg("nblocks"), py::arg("m"), py::arg("n"), py::arg("lda"), py::arg("stride"),
     py::arg("inits"), py::arg("k"), py::arg("l"), py::arg("loops"), py::arg("h"), py::arg("threads") = 1);
  m.def("cur_reconstruct", [](const FArray& A, const std::vector<Index>& I, const std::vector<Index>& J,
                              const FArray& U) {
    Matrix M = from_np(A);
    CurDecomposition c{mkset(I, M.rows()), mkset(J, M.cols()), from_np(U), 0};
    return to_np(cur_reconstruct(M, c));
  });
  m.def("cur_evaluate", [](const FArray& A, const std::vector<Index>& I, const std::vector<Index>& J,
                           const FArray& U, const std::string& norm) {
    Matrix M = from_np(A);
    CurDecomposition c{mkset(I, M.rows()), mkset(J, M.cols()), from_np(U), 0};
    NormKind k = norm == "spectral" ? NormKind::Spectral : norm == "chebyshev" ? NormKind::Chebyshev : NormKind::Frobenius;
    return cur_evaluate(M, c, k);
  }, py::arg("A"), py::arg("I"), py::arg("J"), py::arg("U"), py::arg("norm") = "frobenius");

  // ---- remaining CUR / LRA entry points (cur.cpp:170-323, linalg.cpp:153-161, lra.cpp:65-86)
  m.def("condition_number", [](const FArray& A, double tol) { return condition_number(from_np(A), tol); },
        py::arg("A"), py::arg("rank_tol") = 1e-10);
  m.def("truncate_rank", [](const FArray& A, Index rho) {
    LowRankFactors f = truncate_rank(from_np(A), rho);
    return py::make_tuple(to_np(f.U), to_np(f.V));
  });
  m.def("cynical_cur", [](const FArray& A, Index p, Index q, Index k, Index l, Index r, Rng& rng) {
    Matrix M = from_np(A);
    DenseOracle o(M);
    return cur_dict(cynical_cur(o, p, q, k, l, r, rng));
  });
  m.def("top_svd_to_cur", [](const FArray& S, const FArray& sigma, const FArray& T, Index k, Index l, double h,
                             const std::string& sel, Rng& rng) {
    Svd f{from_np(S), np_vec(sigma), from_np(T)};
    return cur_dict(top_svd_to_cur(f, k, l, h, sel == "sampled" ? CurSelector::Sampled : CurSelector::Deterministic, rng));
  });
  m.def("lra_to_top_svd3", [](const FArray& A, const FArray& W, const FArray& B, Index r) {
    Svd t = lra_to_top_svd(from_np(A), from_np(W), from_np(B), r);
    return py::make_tuple(to_np(t.S), vec_np(t.sigma), to_np(t.T));
  });
  m.def("deterministic_error_diagnostic", [](const FArray& M, const PyOp& H, Index r) {
    auto [b, a] = deterministic_error_diagnostic(from_np(M), *H.p, r);
    return py::make_tuple(b, a);
  });

  // ---- sketch operators
  py::class_<PyOp>(m, "SketchOperator", py::module_local())
      .def("rows", [](const PyOp& o) { return o.p->rows(); })
      .def("cols", [](const PyOp& o) { return o.p->cols(); })
      .def("kind", [](const PyOp& o) { return o.p->kind(); })
      .def("apply", [](const PyOp& o, const FArray& M) { return to_np(o.p->apply(from_np(M))); })
      .def("apply_transpose", [](const PyOp& o, const FArray& M) { return to_np(o.p->apply_transpose(from_np(M))); });
  m.def("make_permutation", [](std::vector<Index> s) { return PyOp{make_permutation(std::move(s))}; });
  m.def("make_sign_diagonal", [](const FArray& d) { return PyOp{make_sign_diagonal(np_vec(d))}; });
  m.def("make_abridged_hadamard", [](Index n, int d) { return PyOp{make_abridged_hadamard(n, d)}; });
  m.def("make_sparse_circulant", [](Index n, double f, std::vector<std::pair<Index, double>> nz) {
    return PyOp{make_sparse_circulant(n, f, std::move(nz))};
  });
  m.def("make_inverse_bidiagonal", [](const FArray& b, bool lower) { return PyOp{make_inverse_bidiagonal(np_vec(b), lower)}; },
        py::arg("subdiag"), py::arg("lower") = true);
  m.def("gen_inverse_bidiagonal", [](Index n, Rng& r) { return PyOp{gen_inverse_bidiagonal(n, r)}; });
  m.def("gen_householder_chain", [](Index n, Index q, Rng& r) { return PyOp{gen_householder_chain(n, q, r)}; });
  m.def("make_abridged_fourier", [](Index n, int d) { return PyOp{make_abridged_fourier(n, d)}; });
  auto cnp = [](const CMatrix& M) {
    py::array_t<std::complex<double>, py::array::f_style> a({M.rows(), M.cols()});
    auto* p = a.mutable_data();
    for (Index j = 0; j < M.cols(); ++j)
      for (Index i = 0; i < M.rows(); ++i) p[i + j * M.rows()] = {M.re(i, j), M.im(i, j)};
    return a;
  };
  auto npc = [](const py::array_t<std::complex<double>, py::array::f_style | py::array::forcecast>& a) {
    if (a.ndim() != 2) throw std::invalid_argument("expected a 2-D complex array");
    CMatrix M{Matrix(a.shape(0), a.shape(1)), Matrix(a.shape(0), a.shape(1))};
    const auto* p = a.data();
    for (Index j = 0; j < M.cols(); ++j)
      for (Index i = 0; i < M.rows(); ++i) {
        M.re(i, j) = p[i + j * M.rows()].real();
        M.im(i, j) = p[i + j * M.rows()].imag();
      }
    return M;
  };
  m.def("apply_complex", [=](const PyOp& op, const py::array_t<std::complex<double>, py::array::f_style | py::array::forcecast>& M) {
    return cnp(op.p->apply_complex(npc(M)));
  });
  m.def("apply_transpose_complex", [=](const PyOp& op, const py::array_t<std::complex<double>, py::array::f_style | py::array::forcecast>& M) {
    return cnp(op.p->apply_transpose_complex(npc(M)));
  });
  m.def("materialize_complex", [=](const PyOp& op) { return cnp(materialize_complex(*op.p)); });
  m.def("make_sum", [](const std::vector<PyOp>& ops, const std::vector<int>& signs) {
    std::vector<OpPtr> v;
    for (auto& o : ops) v.push_back(o.p);
    return PyOp{make_sum(std::move(v), signs)};
  });
  m.def("gen_scaled_diagonal", [](Index n, Rng& r) { return PyOp{gen_scaled_diagonal(n, r)}; });
  m.def("bidiagonal_factor", [](Index n, const std::vector<int>& s) { return to_np(bidiagonal_factor(n, s)); });
  m.def("gen_bidiagonal_product", [](Index n, Index T, Rng& r, bool st) { return to_np(gen_bidiagonal_product(n, T, r, st)); },
        py::arg("n"), py::arg("T"), py::arg("rng"), py::arg("standardize") = true);
  m.def("bidiagonal_product_column", [](Index n, Index T, Index j, Rng& r) { return vec_np(bidiagonal_product_column(n, T, j, r)); });
  m.def("ks_normality", [](const std::vector<double>& x) { return ks_normality(x); });
  m.def("make_gaussian", [](const FArray& G) { return PyOp{make_gaussian(from_np(G))}; });
  m.def("make_sub_identity", [](const std::vector<Index>& sel, Index total) {
    return PyOp{make_sub_identity(mkset(sel, total), total)};
  });
  m.def("make_product", [](const std::vector<PyOp>& ops) {
    std::vector<OpPtr> v;
    for (auto& o : ops) v.push_back(o.p);
    return PyOp{make_product(std::move(v))};
  });
  m.def("take_columns", [](const PyOp& op, const std::vector<Index>& cols) {
    return PyOp{take_columns(op.p, mkset(cols, op.p->cols()))};
  });
  m.def("take_columns_random", [](const PyOp& op, Index l, Rng& rng) {
    return PyOp{take_columns(op.p, l, ColumnMode::Random, rng)};
  });
  m.def("gen_permutation", [](Index n, Rng& r) { return PyOp{gen_permutation(n, r)}; });
  m.def("gen_sign_diagonal", [](Index n, Rng& r) { return PyOp{gen_sign_diagonal(n, r)}; });
  m.def("gen_sparse_circulant", [](Index n, Index s, Rng& r) { return PyOp{gen_sparse_circulant(n, s, r)}; });
  m.def("gen_gaussian", [](Index a, Index b, Rng& r) { return PyOp{gen_gaussian(a, b, r)}; });
  m.def("gen_aph", [](Index n, int d, Rng& r) { return PyOp{gen_aph(n, d, r)}; });
  m.def("gen_asph", [](Index n, int d, Rng& r, bool scaled) { return PyOp{gen_asph(n, d, r, scaled)}; },
        py::arg("n"), py::arg("d"), py::arg("rng"), py::arg("scaled_diag") = false);
  m.def("apply", [](const PyOp& op, const FArray& M, const std::string& side) {
    return to_np(apply(*op.p, from_np(M), side == "right" ? Side::Right : Side::Left));
  });
  m.def("materialize", [](const PyOp& op) { return to_np(materialize(*op.p)); });
  m.def("reset_op_counter", &reset_op_counter);
  m.def("op_counter", []() { return py::make_tuple(op_counter().adds, op_counter().muls); });

  // ---- lra
  m.def("range_finder", [](const FArray& M, const PyOp& H, Index r, bool truncated) {
    LowRankFactors f = range_finder(from_np(M), *H.p, r, truncated ? RangeVariant::TruncatedRankR : RangeVariant::BasisQr);
    return py::make_tuple(to_np(f.U), to_np(f.V));
  }, py::arg("M"), py::arg("H"), py::arg("r"), py::arg("truncated") = false);
  // ||M - U V||_F (slra_cli.cpp:286 error, Frobenius as in north_star)
  m.def("lowrank_residual_frobenius", [](const FArray& M, const FArray& U, const FArray& V) {
    return frobenius_norm(sub(from_np(M), matmul(from_np(U), from_np(V))));
  });
  m.def("lra_premult", [](const FArray& M, const PyOp& F, const PyOp& H, Index r, bool truncated) {
    LowRankFactors f = lra_premult(from_np(M), *F.p, *H.p, r,
                                   truncated ? RangeVariant::TruncatedRankR : RangeVariant::BasisQr);
    return py::make_tuple(to_np(f.U), to_np(f.V));
  }, py::arg("M"), py::arg("F"), py::arg("H"), py::arg("r"), py::arg("truncated") = false);
  m.def("two_stage_truncate", [](const FArray& U, const FArray& V, Index r) {
    LowRankFactors f{from_np(U), from_np(V), 0};
    LowRankFactors g = two_stage_truncate(f, r);
    return py::make_tuple(to_np(g.U), to_np(g.V));
  });
  m.def("posterior_error_estimate", [](const FArray& M, const FArray& U, const FArray& V, Index q, Index s, Rng& rng) {
    Matrix A = from_np(M);
    DenseOracle o(A);
    LowRankFactors f{from_np(U), from_np(V), 0};
    LraErrorEstimate e = posterior_error_estimate(o, f, q, s, rng);
    return py::make_tuple(e.estimate_frobenius, e.ci_lo, e.ci_hi, e.has_interval);
  });

  // ---- leverage (leverage.hpp)
  auto scores_from = [](const FArray& p, double beta, Index r) {
    LeverageScores s;
    s.p = np_vec(p);
    s.beta = beta;
    s.r = r;
    return s;
  };
  auto sr_dict = [](const SampleRescale& s) {
    py::dict d;
    d["indices"] = s.indices;
    d["d"] = vec_np(s.d);
    return d;
  };
  m.def("svd_leverage_scores", [](const FArray& T, double beta) {
    LeverageScores s = svd_leverage_scores(from_np(T), beta);
    return py::make_tuple(vec_np(s.p), s.beta, s.r);
  }, py::arg("T"), py::arg("beta") = 1.0);
  m.def("sample_exactly", [=](const FArray& p, Index l, Rng& rng) { return sr_dict(sample_exactly(scores_from(p, 1.0, 1), l, rng)); });
  m.def("sample_expected", [=](const FArray& p, Index l, Rng& rng) { return sr_dict(sample_expected(scores_from(p, 1.0, 1), l, rng)); });
  m.def("collapse_duplicates", [=](const std::vector<Index>& idx, const FArray& d) {
    SampleRescale s;
    s.indices = idx;
    s.d = np_vec(d);
    return sr_dict(collapse_duplicates(s));
  });
  m.def("cur_via_leverage", [=](const FArray& M, Index r, Index k, Index l, double beta, double beta_bar,
                                const std::string& mode, std::optional<FArray> scores, Rng& rng, bool plain) {
    Matrix A = from_np(M);
    DenseOracle o(A);
    std::optional<LeverageScores> sc;
    if (scores) sc = scores_from(*scores, beta, r);
    CurDecomposition c = cur_via_leverage(o, r, k, l, beta, beta_bar,
                                          mode == "exactly" ? SampleMode::Exactly : SampleMode::Expected, sc, rng, plain);
    return cur_dict(c);
  }, py::arg("M"), py::arg("r"), py::arg("k"), py::arg("l"), py::arg("beta"), py::arg("beta_bar"), py::arg("mode"),
     py::arg("scores"), py::arg("rng"), py::arg("plain_nucleus") = false);
  m.def("lra_to_top_svd", [](const FArray& U, const FArray& V, Index r) {
    LowRankFactors f{from_np(U), from_np(V), 0};
    Svd t = lra_to_top_svd(f, r);
    return py::make_tuple(to_np(t.S), vec_np(t.sigma), to_np(t.T));
  });
  m.def("refine_lra", [](const FArray& M, const FArray& U, const FArray& V, Index target, Index r, Index k, Index l,
                         Rng& rng) {
    Matrix A = from_np(M);
    DenseOracle o(A);
    LowRankFactors f{from_np(U), from_np(V), target};
    return cur_dict(refine_lra(o, f, r, k, l, rng));
  });
  m.def("uniform_scores", [](Index n) { return vec_np(uniform_scores(n).p); });
  m.def("gaussian_score_gap", [](const FArray& G) { return gaussian_score_gap(from_np(G)); });
  m.def("sample_bound_quadratic", &sample_bound_quadratic);
  m.def("sample_bound_loglinear", &sample_bound_loglinear);
  m.def("epsilon_for_sample", &epsilon_for_sample);

  // ---- hss (hss.hpp:44-52)
  m.def("build_hss", [](const FArray& M, int L, Index r, double tol, const std::string& strategy, Rng& rng) {
    Matrix A = from_np(M);
    DenseOracle o(A);
    if (strategy != "svd" && strategy != "cur_ca") throw std::invalid_argument("strategy: svd | cur_ca");
    HssMatrix h = build_hss(o, L, r, tol, strategy == "svd" ? HssStrategy::Svd : HssStrategy::CurCa, rng);
    py::dict d = hss_dict(h);
    d["accesses"] = o.accesses();
    return d;
  });
  m.def("hss_matvec", [](const py::dict& h, const FArray& x) { return vec_np(hss_matvec(hss_from(h), np_vec(x))); });
  m.def("hss_reconstruct", [](const py::dict& h) { return to_np(hss_reconstruct(hss_from(h))); });
  m.def("hss_error", [](const py::dict& h, const FArray& M, const std::string& norm) {
    const NormKind k = norm == "spectral" ? NormKind::Spectral : norm == "chebyshev" ? NormKind::Chebyshev
                                                                                      : NormKind::Frobenius;
    return hss_error(hss_from(h), from_np(M), k);
  });

  // ---- lsr
  m.def("sketch_solve", [](const FArray& A, const FArray& b, const PyOp& F, bool with_true) {
    LsrProblem p{from_np(A), np_vec(b)};
    LsrReport r = sketch_solve(p, *F.p, with_true);
    py::dict d;
    d["x_hat"] = vec_np(r.x_hat);
    d["sketched_residual"] = r.sketched_residual;
    d["true_residual"] = r.true_residual;
    d["ratio"] = r.ratio;
    d["k"] = r.k;
    return d;
  }, py::arg("A"), py::arg("b"), py::arg("F"), py::arg("with_true_residual") = false);
  m.def("solve_with_retries", [](const FArray& A, const FArray& b, const PyOp& F, const std::vector<PyOp>& qf,
                                 int max_retries, double accept_tol, Rng& rng) {
    LsrProblem p{from_np(A), np_vec(b)};
    std::vector<OpPtr> q;
    for (auto& o : qf) q.push_back(o.p);
    LsrReport r = solve_with_retries(p, F.p, q, max_retries, accept_tol, rng);
    py::dict d;
    d["x_hat"] = vec_np(r.x_hat);
    d["sketched_residual"] = r.sketched_residual;
    d["k"] = r.k;
    d["validated"] = r.validated;
    d["attempts"] = r.attempts;
    return d;
  });
  m.def("solve_exact", [](const FArray& A, const FArray& b) {
    return vec_np(solve_exact(LsrProblem{from_np(A), np_vec(b)}));
  });
  m.def("residual_norm", [](const FArray& A, const FArray& b, const FArray& x) {
    return residual_norm(LsrProblem{from_np(A), np_vec(b)}, np_vec(x));
  });
  m.def("residual_ratio", [](const FArray& A, const FArray& b, const FArray& x) {
    return residual_ratio(LsrProblem{from_np(A), np_vec(b)}, np_vec(x));
  });

  // ---- testgen
  m.def("random_orthonormal", [](Index r, Index c, Rng& rng) { return to_np(random_orthonormal(r, c, rng)); });
  m.def("gen_svd_profile", [](Index n, Index r, Rng& rng) { return to_np(gen_svd_profile(n, r, rng)); });
  m.def("gen_factor_gaussian", [](Index mm, Index n, Index r, double noise, Rng& rng) {
    return to_np(gen_factor_gaussian(mm, n, r, noise, rng));
  });
  m.def("gen_lsr_gaussian", [](Index mm, Index n, double noise, Rng& rng) {
    LsrProblem p = gen_lsr_gaussian(mm, n, noise, rng);
    return py::make_tuple(to_np(p.A), vec_np(p.b));
  });
}
