// Python binding of the C++ host layer (namespace slra). Host-array entry
// points mirror the reference signatures; *_device entry points take raw
// device pointers (e.g. torch tensor.data_ptr()) for HBM-resident runs.
#include <chrono>
#include <mutex>
#include <unordered_map>

#include <pybind11/complex.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "slra/cur.hpp"
#include "slra/devbuf.hpp"
#include "slra/device.hpp"
#include "slra/errors.hpp"
#include "slra/hss.hpp"
#include "slra/leverage.hpp"
#include "slra/lra.hpp"
#include "slra/lsr.hpp"
#include "slra/sketch.hpp"
#include "slra/testgen.hpp"

namespace py = pybind11;
using namespace slra;

using FArray = py::array_t<double, py::array::f_style | py::array::forcecast>;

static Matrix from_np(const FArray& a) {
  if (a.ndim() == 1) {
    Matrix M(a.shape(0), 1);
    std::copy(a.data(), a.data() + a.shape(0), M.data());
    return M;
  }
  if (a.ndim() != 2) throw std::invalid_argument("expected a 1-D or 2-D array");
  Matrix M(a.shape(0), a.shape(1));
  std::copy(a.data(), a.data() + M.size(), M.data());
  return M;
}
static FArray to_np(const Matrix& M) {
  FArray a({M.rows(), M.cols()});
  std::copy(M.data(), M.data() + M.size(), a.mutable_data());
  return a;
}
// Result arrays of the host-buffer entry points, backed by page-locked
// blocks: the D2H copy lands in the returned array at the link's rate (no
// pageable staging, no second host copy). A block returns to a free list
// keyed by size when its array dies, so steady-state calls allocate nothing.
static std::mutex pin_mu;
static std::unordered_multimap<size_t, void*>* pin_free = new std::unordered_multimap<size_t, void*>();
static size_t pin_free_bytes = 0;
constexpr size_t kPinPoolCap = size_t(1) << 30;  // page-locked bytes kept for reuse
// HBM staging buffers of the host-buffer entry points (one per entry),
// released through the old context when set_device replaces it
static DeviceMatrix* g_staging = new DeviceMatrix[4];
static DeviceMatrix& staging(int slot, Index rows, Index cols) {
  DeviceMatrix& s = g_staging[slot];
  if (s.rows() != rows || s.cols() != cols) s = DeviceMatrix(rows, cols);
  return s;
}
static void release_staging() {
  for (int i = 0; i < 4; ++i) g_staging[i] = DeviceMatrix();
}
static FArray pinned_np(Index rows, Index cols) {
  const size_t bytes = sizeof(double) * static_cast<size_t>(rows) * static_cast<size_t>(cols);
  void* p = nullptr;
  {
    std::lock_guard<std::mutex> g(pin_mu);
    auto it = pin_free->find(bytes);
    if (it != pin_free->end()) {
      p = it->second;
      pin_free->erase(it);
      pin_free_bytes -= bytes;
    }
  }
  if (!p) check(slra_host_alloc(static_cast<int64_t>(bytes ? bytes : 8), &p), "pinned result buffer");
  py::capsule hold(new std::pair<void*, size_t>(p, bytes), [](void* h) {
    auto* ph = static_cast<std::pair<void*, size_t>*>(h);
    bool keep = false;
    {
      std::lock_guard<std::mutex> g(pin_mu);
      if (pin_free_bytes + ph->second <= kPinPoolCap) {  // bounded: beyond the cap, give it back
        pin_free->emplace(ph->second, ph->first);
        pin_free_bytes += ph->second;
        keep = true;
      }
    }
    if (!keep) slra_host_free(ph->first);
    delete ph;
  });
  return FArray({rows, cols}, {static_cast<py::ssize_t>(sizeof(double)), static_cast<py::ssize_t>(sizeof(double) * rows)},
                static_cast<double*>(p), hold);
}
static FArray download_pinned(const DeviceMatrix& M) {
  if (M.ld() != M.rows()) return to_np(M.download());
  FArray a = pinned_np(M.rows(), M.cols());
  check(slra_memcpy_d2h(device_context(), a.mutable_data(), M.data(), 8 * M.rows() * M.cols()), "download");
  return a;
}
static py::array_t<double> vec_np(const Vector& v) {
  py::array_t<double> a(static_cast<py::ssize_t>(v.size()));
  std::copy(v.begin(), v.end(), a.mutable_data());
  return a;
}
static Vector np_vec(const FArray& a) { return Vector(a.data(), a.data() + a.size()); }
static IndexSet mkset(const std::vector<Index>& v, Index bound) { return IndexSet(v, bound); }
struct PyOp {
  OpPtr p;
};
template <typename T>
static T* ptr(uintptr_t p) {
  return reinterpret_cast<T*>(p);
}

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

static NormKind norm_kind(const std::string& s) {
  if (s == "spectral") return NormKind::Spectral;
  if (s == "frobenius") return NormKind::Frobenius;
  if (s == "chebyshev") return NormKind::Chebyshev;
  throw std::invalid_argument("norm: spectral | frobenius | chebyshev");
}

static py::dict cur_dict(const CurDecomposition& c) {
  py::dict d;
  d["I"] = c.row_set.indices();
  d["J"] = c.col_set.indices();
  d["nucleus"] = to_np(c.nucleus);
  d["r"] = c.r;
  if (c.tsig.cols() > 0) {
    d["tsig"] = to_np(c.tsig);
    d["sr"] = to_np(c.sr);
  }
  return d;
}

static py::dict plan_dict(const SketchPlan& p) {
  py::dict d;
  d["tree"] = p.tree;
  d["width"] = p.width;
  d["count"] = p.count;
  d["src"] = p.src;
  d["coef"] = p.coef;
  d["q"] = p.q;
  return d;
}

PYBIND11_MODULE(_slra, m) {
  m.doc() = "B200 slra hot path: C++ host layer over the sm_100a C-ABI (libslra_cuda.so)";
  auto base = py::register_local_exception<std::runtime_error>(m, "SlraRuntimeError");
  py::register_local_exception<RangeFailure>(m, "RangeFailure", base.ptr());
  py::register_local_exception<SketchRankFailure>(m, "SketchRankFailure", base.ptr());
  py::register_local_exception<PremultRankFailure>(m, "PremultRankFailure", base.ptr());
  py::register_local_exception<SelectionFailure>(m, "SelectionFailure", base.ptr());
  py::register_local_exception<GeneratorRankFailure>(m, "GeneratorRankFailure", base.ptr());
  py::register_local_exception<EmptySample>(m, "EmptySample", base.ptr());
  py::register_local_exception<DeviceError>(m, "DeviceError", base.ptr());

  on_context_release(&release_staging);
  m.def("set_device", [](int dev, uintptr_t stream) { set_device(dev, reinterpret_cast<void*>(stream)); },
        py::arg("device") = 0, py::arg("stream") = 0);
  m.def("launch_count", []() { return slra_ctx_launch_count(device_context()); });
  m.def("set_timing", [](bool on) { check(slra_ctx_set_timing(device_context(), on ? 1 : 0), "set_timing"); });
  m.def("timing_report", []() {
    std::vector<char> buf(1 << 16);
    check(slra_ctx_timing_report(device_context(), buf.data(), (int64_t)buf.size()), "timing_report");
    py::dict d;
    std::string s(buf.data());
    size_t pos = 0;
    while (pos < s.size()) {
      size_t end = s.find(';', pos);
      if (end == std::string::npos) end = s.size();
      const std::string item = s.substr(pos, end - pos);
      const size_t eq = item.find('='), comma = item.find(',');
      if (eq != std::string::npos && comma != std::string::npos)
        d[py::str(item.substr(0, eq))] = py::make_tuple(std::stod(item.substr(eq + 1, comma - eq - 1)),
                                                        std::stoll(item.substr(comma + 1)));
      pos = end + 1;
    }
    return d;
  });
  m.def("stream_ptr", []() { return reinterpret_cast<uintptr_t>(slra_ctx_stream(device_context())); });
  m.def("synchronize", []() { check(slra_ctx_synchronize(device_context()), "synchronize"); });

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
  m.def("chebyshev_norm", [](const FArray& A) { return chebyshev_norm(from_np(A)); });
  m.def("matrix_norm", [](const FArray& A, const std::string& k) { return matrix_norm(from_np(A), norm_kind(k)); });

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
    py::dict d = cur_dict(c);
    d["accesses"] = o.accesses();
    return d;
  }, py::arg("M"), py::arg("r"), py::arg("k"), py::arg("l"), py::arg("beta"), py::arg("beta_bar"), py::arg("mode"),
     py::arg("scores"), py::arg("rng"), py::arg("plain_nucleus") = false);
  m.def("lra_to_top_svd", [](const FArray& U, const FArray& V, Index r) {
    LowRankFactors f;
    f.U = from_np(U);
    f.V = from_np(V);
    Svd t = lra_to_top_svd(f, r);
    return py::make_tuple(to_np(t.S), vec_np(t.sigma), to_np(t.T));
  });
  m.def("refine_lra", [](const FArray& M, const FArray& U, const FArray& V, Index target, Index r, Index k, Index l,
                         Rng& rng) {
    Matrix A = from_np(M);
    DenseOracle o(A);
    LowRankFactors f;
    f.U = from_np(U);
    f.V = from_np(V);
    f.target_rank = target;
    return cur_dict(refine_lra(o, f, r, k, l, rng));
  });
  m.def("uniform_scores", [](Index n) { return vec_np(uniform_scores(n).p); });
  m.def("gaussian_score_gap", [](const FArray& G) { return gaussian_score_gap(from_np(G)); });
  m.def("sample_bound_quadratic", &sample_bound_quadratic);
  m.def("sample_bound_loglinear", &sample_bound_loglinear);
  m.def("epsilon_for_sample", &epsilon_for_sample);

  // ---- hss (hss.hpp:44-52)
  m.def("build_hss", [](const FArray& M, int L, Index r, double tol, const std::string& strategy, Rng& rng) {
    if (strategy != "svd" && strategy != "cur_ca") throw std::invalid_argument("strategy: svd | cur_ca");
    Matrix A = from_np(M);
    DenseOracle o(A);
    HssMatrix h = build_hss(o, L, r, tol, strategy == "svd" ? HssStrategy::Svd : HssStrategy::CurCa, rng);
    py::dict d = hss_dict(h);
    d["accesses"] = o.accesses();
    return d;
  });
  m.def("hss_matvec", [](const py::dict& h, const FArray& x) { return vec_np(hss_matvec(hss_from(h), np_vec(x))); });
  m.def("hss_reconstruct", [](const py::dict& h) { return to_np(hss_reconstruct(hss_from(h))); });
  m.def("hss_error", [](const py::dict& h, const FArray& M, const std::string& norm) {
    return hss_error(hss_from(h), from_np(M), norm_kind(norm));
  });
  m.def("hss_serialize", [](const py::dict& h) { return hss_from(h).serialize(); });
  m.def("hss_deserialize", [](const std::string& s) { return hss_dict(HssMatrix::deserialize(s)); });
  // device-resident: build once, multiply a batch of HBM vectors (bench)
  m.def("hss_matvec_timed", [](const FArray& M, int L, Index r, double tol, const std::string& strategy, Rng& rng,
                               uintptr_t d_x, uintptr_t d_y, int reps) {
    Matrix A = from_np(M);
    DenseOracle o(A);
    HssDevice h = build_hss_device(o, L, r, tol, strategy == "svd" ? HssStrategy::Svd : HssStrategy::CurCa, rng);
    hss_matvec_device(h, ptr<double>(d_x), ptr<double>(d_y));  // warm-up
    check(slra_ctx_synchronize(device_context()), "hss_matvec_timed");
    const auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < reps; ++t) hss_matvec_device(h, ptr<double>(d_x), ptr<double>(d_y));
    check(slra_ctx_synchronize(device_context()), "hss_matvec_timed");
    // seconds per product over the loop (device-resident x, y and generators)
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
  });

  // ---- cur
  m.def("t_factor", &t_factor);
  m.def("maxvol_rows", [](const FArray& A, double h, Index ms) { return maxvol_rows(from_np(A), h, ms).indices(); },
        py::arg("A"), py::arg("h") = 1.1, py::arg("max_swaps") = 0);
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
  m.def("cod_pinv_device", [](uintptr_t G, Index ldg, Index k, Index l, double threshold, uintptr_t P, Index ldp) {
    int64_t rank = 0;
    check(slra_cod_pinv(device_context(), ptr<double>(G), ldg, k, l, threshold, ptr<double>(P), ldp, &rank),
          "cod_pinv");
    return rank;
  });
  m.def("cross_approx", [](const FArray& A, Index r, Index k, Index l, const std::vector<Index>& init_rows, int loops,
                           double h, Rng& rng, std::optional<double> stop_tol) {
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
      if (s.error_estimate) sd["error_estimate"] = *s.error_estimate;
      else sd["error_estimate"] = py::none();
      steps.append(sd);
    }
    d["trace"] = steps;
    d["accesses"] = o.accesses();
    return d;
  }, py::arg("A"), py::arg("r"), py::arg("k"), py::arg("l"), py::arg("init_rows"), py::arg("loops"), py::arg("h"),
     py::arg("rng"), py::arg("stop_tol") = py::none());
  m.def("cur_evaluate", [](const FArray& A, const std::vector<Index>& I, const std::vector<Index>& J,
                           const FArray& U, const std::string& norm) {
    Matrix M = from_np(A);
    CurDecomposition c{mkset(I, M.rows()), mkset(J, M.cols()), from_np(U), 0, false};
    return cur_evaluate(M, c, norm_kind(norm));
  }, py::arg("A"), py::arg("I"), py::arg("J"), py::arg("U"), py::arg("norm") = "frobenius");
  // ---- remaining CUR / LRA entry points (cur.cpp:170-323, linalg.cpp:100-161, lra.cpp:65-127)
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
  m.def("posterior_error_estimate", [](const FArray& M, const FArray& U, const FArray& V, Index q, Index s, Rng& rng) {
    Matrix A = from_np(M);
    DenseOracle o(A);
    LowRankFactors f;
    f.U = from_np(U);
    f.V = from_np(V);
    LraErrorEstimate e = posterior_error_estimate(o, f, q, s, rng);
    return py::make_tuple(e.estimate_frobenius, e.ci_lo, e.ci_hi, e.has_interval);
  });
  m.def("deterministic_error_diagnostic", [](const FArray& M, const PyOp& H, Index r) {
    auto [b, a] = deterministic_error_diagnostic(from_np(M), *H.p, r);
    return py::make_tuple(b, a);
  });
  m.def("cur_evaluate_factored", [](const FArray& A, const std::vector<Index>& I, const std::vector<Index>& J,
                                    const FArray& T, const FArray& S) {
    Matrix M = from_np(A);
    CurDecomposition c{mkset(I, M.rows()), mkset(J, M.cols()), Matrix(), 0, false};
    c.tsig = from_np(T);
    c.sr = from_np(S);
    c.r = c.tsig.cols();
    return cur_evaluate(M, c, NormKind::Frobenius);
  });
  m.def("cur_reconstruct", [](const FArray& A, const std::vector<Index>& I, const std::vector<Index>& J,
                              const FArray& U) {
    Matrix M = from_np(A);
    CurDecomposition c{mkset(I, M.rows()), mkset(J, M.cols()), from_np(U), 0, false};
    return to_np(cur_reconstruct(M, c));
  });

  // ---- sketch operators
  py::class_<PyOp>(m, "SketchOperator", py::module_local())
      .def("rows", [](const PyOp& o) { return o.p->rows(); })
      .def("cols", [](const PyOp& o) { return o.p->cols(); })
      .def("kind", [](const PyOp& o) { return o.p->kind(); })
      .def("apply", [](const PyOp& o, const FArray& M) { return to_np(o.p->apply(from_np(M))); })
      .def("apply_transpose", [](const PyOp& o, const FArray& M) { return to_np(o.p->apply_transpose(from_np(M))); })
      .def("plan", [](const PyOp& o, const std::string& side) {
        return plan_dict(compile_plan(*o.p, side == "right" ? Side::Right : Side::Left));
      });
  m.def("make_permutation", [](std::vector<Index> s) { return PyOp{make_permutation(std::move(s))}; });
  m.def("make_sign_diagonal", [](const FArray& d) { return PyOp{make_sign_diagonal(np_vec(d))}; });
  m.def("make_abridged_hadamard", [](Index n, int d) { return PyOp{make_abridged_hadamard(n, d)}; });
  m.def("make_sparse_circulant", [](Index n, double f, std::vector<std::pair<Index, double>> nz) {
    return PyOp{make_sparse_circulant(n, f, std::move(nz))};
  });
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
  m.def("make_inverse_bidiagonal", [](const FArray& b, bool lower) { return PyOp{make_inverse_bidiagonal(np_vec(b), lower)}; },
        py::arg("subdiag"), py::arg("lower") = true);
  m.def("gen_inverse_bidiagonal", [](Index n, Rng& r) { return PyOp{gen_inverse_bidiagonal(n, r)}; });
  m.def("gen_householder_chain", [](Index n, Index q, Rng& r) { return PyOp{gen_householder_chain(n, q, r)}; });
  m.def("make_abridged_fourier", [](Index n, int d) { return PyOp{make_abridged_fourier(n, d)}; });
  using CArray = py::array_t<std::complex<double>, py::array::f_style | py::array::forcecast>;
  auto cnp = [](const CMatrix& M) {
    py::array_t<std::complex<double>, py::array::f_style> a({M.rows(), M.cols()});
    auto* p = a.mutable_data();
    for (Index j = 0; j < M.cols(); ++j)
      for (Index i = 0; i < M.rows(); ++i) p[i + j * M.rows()] = {M.re(i, j), M.im(i, j)};
    return a;
  };
  auto npc = [](const CArray& a) {
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
  m.def("apply_complex", [=](const PyOp& op, const CArray& M) { return cnp(op.p->apply_complex(npc(M))); });
  m.def("apply_transpose_complex", [=](const PyOp& op, const CArray& M) {
    return cnp(op.p->apply_transpose_complex(npc(M)));
  });
  m.def("materialize_complex", [=](const PyOp& op) { return cnp(materialize_complex(*op.p)); });
  m.def("make_gaussian", [](const FArray& G) { return PyOp{make_gaussian(from_np(G))}; });
  m.def("gen_gaussian", [](Index a, Index b, Rng& r) { return PyOp{gen_gaussian(a, b, r)}; });
  m.def("gen_permutation", [](Index n, Rng& r) { return PyOp{gen_permutation(n, r)}; });
  m.def("gen_sign_diagonal", [](Index n, Rng& r) { return PyOp{gen_sign_diagonal(n, r)}; });
  m.def("gen_sparse_circulant", [](Index n, Index s, Rng& r) { return PyOp{gen_sparse_circulant(n, s, r)}; });
  m.def("gen_aph", [](Index n, int d, Rng& r) { return PyOp{gen_aph(n, d, r)}; });
  m.def("gen_asph", [](Index n, int d, Rng& r, bool scaled) { return PyOp{gen_asph(n, d, r, scaled)}; },
        py::arg("n"), py::arg("d"), py::arg("rng"), py::arg("scaled_diag") = false);
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
  m.def("ks_normality", [](const std::vector<double>& x) {
    KsResult k = ks_normality(x);
    return py::make_tuple(k.statistic, k.pass);
  });
  m.def("apply", [](const PyOp& op, const FArray& M, const std::string& side) {
    return to_np(apply(*op.p, from_np(M), side == "right" ? Side::Right : Side::Left));
  });
  m.def("materialize", [](const PyOp& op) { return to_np(materialize(*op.p)); });

  // ---- lra / lsr
  m.def("range_finder", [](const FArray& M, const PyOp& H, Index r, bool truncated) {
    LowRankFactors f = range_finder(from_np(M), *H.p, r, truncated ? RangeVariant::TruncatedRankR : RangeVariant::BasisQr);
    return py::make_tuple(to_np(f.U), to_np(f.V));
  }, py::arg("M"), py::arg("H"), py::arg("r"), py::arg("truncated") = false);
  m.def("lra_premult", [](const FArray& M, const PyOp& F, const PyOp& H, Index r, bool truncated) {
    LowRankFactors f = lra_premult(from_np(M), *F.p, *H.p, r,
                                   truncated ? RangeVariant::TruncatedRankR : RangeVariant::BasisQr);
    return py::make_tuple(to_np(f.U), to_np(f.V));
  }, py::arg("M"), py::arg("F"), py::arg("H"), py::arg("r"), py::arg("truncated") = false);
  m.def("two_stage_truncate", [](const FArray& U, const FArray& V, Index r) {
    LowRankFactors f;
    f.U = from_np(U);
    f.V = from_np(V);
    f.target_rank = f.U.cols();
    LowRankFactors g = two_stage_truncate(f, r);
    return py::make_tuple(to_np(g.U), to_np(g.V));
  });
  m.def("solve_with_retries", [](const FArray& A, const FArray& b, const PyOp& F, const std::vector<PyOp>& qf,
                                 int max_retries, double accept_tol, Rng& rng) {
    std::vector<OpPtr> q;
    for (auto& o : qf) q.push_back(o.p);
    LsrReport r = solve_with_retries(LsrProblem{from_np(A), np_vec(b)}, F.p, q, max_retries, accept_tol, rng);
    py::dict d;
    d["x_hat"] = vec_np(r.x_hat);
    d["sketched_residual"] = r.sketched_residual;
    d["k"] = r.k;
    d["validated"] = r.validated;
    d["attempts"] = r.attempts;
    return d;
  });
  m.def("sketch_solve", [](const FArray& A, const FArray& b, const PyOp& F, bool with_true) {
    LsrReport rep = sketch_solve(LsrProblem{from_np(A), np_vec(b)}, *F.p, with_true);
    py::dict d;
    d["x_hat"] = vec_np(rep.x_hat);
    d["sketched_residual"] = rep.sketched_residual;
    d["true_residual"] = rep.true_residual;
    d["ratio"] = rep.ratio;
    d["k"] = rep.k;
    return d;
  }, py::arg("A"), py::arg("b"), py::arg("F"), py::arg("with_true_residual") = false);
  m.def("solve_exact", [](const FArray& A, const FArray& b) { return vec_np(solve_exact(LsrProblem{from_np(A), np_vec(b)})); });
  m.def("residual_norm", [](const FArray& A, const FArray& b, const FArray& x) {
    return residual_norm(LsrProblem{from_np(A), np_vec(b)}, np_vec(x));
  });
  m.def("residual_ratio", [](const FArray& A, const FArray& b, const FArray& x) {
    return residual_ratio(LsrProblem{from_np(A), np_vec(b)}, np_vec(x));
  });

  // ---- testgen
  m.def("gen_factor_gaussian", [](Index mm, Index n, Index r, double noise, Rng& rng) {
    return to_np(gen_factor_gaussian(mm, n, r, noise, rng));
  });
  m.def("gen_lsr_gaussian", [](Index mm, Index n, double noise, Rng& rng) {
    LsrProblem p = gen_lsr_gaussian(mm, n, noise, rng);
    return py::make_tuple(to_np(p.A), vec_np(p.b));
  });
  m.def("gen_cauchy_block", [](Index mm, Index n, Rng& rng) { return to_np(gen_cauchy_block(mm, n, rng)); });
  m.def("gen_log_kernel_block", [](Index mm, Index n, Rng& rng) { return to_np(gen_log_kernel_block(mm, n, rng)); });

  // ---- end-to-end form of range_finder(M, H, r, variant) (lra.hpp): M read
  // straight from the caller's (pinned) host buffer, U/V returned to the host.
  m.def("range_finder_host", [](uintptr_t M_host, Index mm, Index n, const PyOp& H, Index r, bool truncated) {
    const SketchPlan plan = compile_plan(*H.p, Side::Right);
    DeviceMatrix& dM = staging(0, mm, n);
    check(slra_memcpy_h2d(device_context(), dM.data(), reinterpret_cast<const void*>(M_host), 8 * mm * n),
          "range_finder_host");
    const Index uc = truncated ? r : H.p->cols();
    DeviceMatrix dU(mm, uc), dV(uc, n);
    DevBuf<double> out(2);
    range_finder_device(dM, plan, r, truncated ? RangeVariant::TruncatedRankR : RangeVariant::BasisQr, dU, dV,
                        out.get());
    auto o = out.download();
    return py::make_tuple(to_np(dU.download()), to_np(dV.download()), o[0], o[1]);
  });

  // ---- end-to-end range_finder(M, H_s, r, variant) for several sketches of
  // the same M: M crosses the bus once, the factorisations of all sketches
  // run batched on the device, every (U_s, V_s, resid_s, norm_s) comes back.
  m.def("range_finder_batched_host", [](uintptr_t M_host, Index mm, Index n, const std::vector<PyOp>& Hs, Index r,
                                        bool truncated) {
    const int nsk = static_cast<int>(Hs.size());
    if (nsk < 1) throw std::invalid_argument("range_finder_batched_host: no sketches");
    const Index l = Hs[0].p->cols();
    DeviceMatrix* staging = &::staging(1, mm, n);  // reused HBM staging buffer
    check(slra_memcpy_h2d(device_context(), staging->data(), reinterpret_cast<const void*>(M_host), 8 * mm * n),
          "range_finder_batched_host");
    std::vector<SketchPlan> plans;
    std::vector<DevBuf<int64_t>> dsrc;
    std::vector<DevBuf<double>> dcoef;
    std::vector<DevBuf<int32_t>> dq;
    std::vector<const int64_t*> src(nsk);
    std::vector<const double*> coef(nsk);
    std::vector<const int32_t*> q(nsk);
    std::vector<int64_t> width(nsk);
    std::vector<int> tree(nsk);
    const Index uc = truncated ? r : l;
    std::vector<DeviceMatrix> dU, dV;
    std::vector<double*> Up(nsk), Vp(nsk);
    for (int s = 0; s < nsk; ++s) {
      if (Hs[s].p->rows() != n || Hs[s].p->cols() != l) throw std::invalid_argument("range_finder_batched_host: H");
      plans.push_back(compile_plan(*Hs[s].p, Side::Right));
      dsrc.emplace_back(plans.back().src);
      dcoef.emplace_back(plans.back().coef);
      dq.emplace_back(plans.back().q);
      dU.emplace_back(mm, uc);
      dV.emplace_back(uc, n);
    }
    for (int s = 0; s < nsk; ++s) {
      src[s] = dsrc[s].get();
      coef[s] = dcoef[s].get();
      q[s] = dq[s].get();
      width[s] = plans[s].width;
      tree[s] = plans[s].tree;
      Up[s] = dU[s].data();
      Vp[s] = dV[s].data();
    }
    DevBuf<double> out(2 * static_cast<size_t>(nsk));
    std::vector<int32_t> status(nsk, 0);
    check(slra_range_finder_batched(device_context(), staging->data(), mm, mm, n, nsk, src.data(), coef.data(),
                                    q.data(), width.data(), tree.data(), l, r, truncated ? 1 : 0, Up.data(), mm,
                                    Vp.data(), uc, out.get(), nullptr, status.data()),
          "range_finder_batched_host");
    for (int s = 0; s < nsk; ++s) check(status[s], "range_finder_batched_host");
    const auto o = out.download();
    py::list res;
    for (int s = 0; s < nsk; ++s)
      res.append(py::make_tuple(download_pinned(dU[s]), download_pinned(dV[s]), o[2 * s], o[2 * s + 1]));
    return res;
  });

  // ---- end-to-end sketch_solve(p, F, false) + residual_norm(p, x_hat)
  // (lsr.hpp) with A (m x d, column-major) and b read from the caller's
  // (pinned) host buffers; x_hat and both residuals come back to the host.
  m.def("sketch_solve_host", [](uintptr_t A_host, uintptr_t b_host, Index mm, Index d, const PyOp& F) {
    const SketchPlan plan = compile_plan(*F.p, Side::Left);
    DeviceMatrix* staging = &::staging(3, mm, d + 1);  // reused HBM staging buffer
    slra_ctx cx = device_context();
    double* dA = staging->data();
    double* db = dA + mm * d;
    check(slra_memcpy_h2d(cx, dA, reinterpret_cast<const void*>(A_host), 8 * mm * d), "sketch_solve_host");
    check(slra_memcpy_h2d(cx, db, reinterpret_cast<const void*>(b_host), 8 * mm), "sketch_solve_host");
    DevBuf<int64_t> src(plan.src);
    DevBuf<double> coef(plan.coef);
    DevBuf<int32_t> q(plan.q);
    DevBuf<double> x(static_cast<size_t>(d)), out(2);
    double sres = 0;
    check(slra_sketch_solve(cx, dA, mm, mm, d, db, src.get(), coef.get(), q.get(), plan.width, plan.tree, plan.count,
                            x.get(), &sres),
          "sketch_solve");
    check(slra_lsr_residual(cx, dA, mm, mm, d, db, x.get(), out.get()), "residual_norm");
    Vector xv = x.download();
    return py::make_tuple(vec_np(xv), sres, std::sqrt(out.download()[0]));
  });

  // ---- end-to-end cross_approx(M, ...) + cur_evaluate(M, c, Frobenius)
  // (cur.hpp) with M read from the caller's (pinned) host buffer; I, J, the
  // nucleus and the residual come back to the host.
  m.def("cross_approx_host", [](uintptr_t M_host, Index mm, Index n, Index r, Index k, Index l,
                                const std::vector<Index>& init_rows, int loops, double h) {
    DeviceMatrix* staging = &::staging(2, mm, n);  // reused HBM staging buffer
    check(slra_memcpy_h2d(device_context(), staging->data(), reinterpret_cast<const void*>(M_host), 8 * mm * n),
          "cross_approx_host");
    DeviceOracle o(staging->data(), mm, n, mm);
    Rng rng(0);
    auto [c, trace] = cross_approx(o, r, k, l, mkset(init_rows, mm), loops, h, std::nullopt, rng);
    const double res = cur_evaluate(o, c, NormKind::Frobenius);
    py::dict d = cur_dict(c);
    d["residual"] = res;
    return d;
  });

  // ---- device-resident entry points (raw device pointers)
  m.def("range_finder_device", [](uintptr_t M, Index ldm, Index mm, Index n, const py::dict& plan, Index r,
                                  bool truncated, uintptr_t U, Index ldu, uintptr_t V, Index ldv, uintptr_t out,
                                  uintptr_t src, uintptr_t coef, uintptr_t q) {
    // plan arrays already on the device (src/coef/q pointers); shape from the dict
    check(slra_range_finder(device_context(), ptr<double>(M), ldm, mm, n, ptr<int64_t>(src), ptr<double>(coef),
                            ptr<int32_t>(q), plan["width"].cast<Index>(), plan["tree"].cast<int>(),
                            plan["count"].cast<Index>(), r, truncated ? 1 : 0, ptr<double>(U), ldu, ptr<double>(V), ldv,
                            ptr<double>(out), nullptr),
          "range_finder");
  });
  // nsk sketches of one HBM-resident M in one call: plans = [(width, tree, src_ptr, coef_ptr, q_ptr), ...]
  m.def("range_finder_batched_device", [](uintptr_t M, Index ldm, Index mm, Index n,
                                          const std::vector<std::tuple<Index, int, uintptr_t, uintptr_t, uintptr_t>>& plans,
                                          Index l, Index r, bool truncated, const std::vector<uintptr_t>& U, Index ldu,
                                          const std::vector<uintptr_t>& V, Index ldv, uintptr_t out) {
    const int nsk = static_cast<int>(plans.size());
    std::vector<const int64_t*> src(nsk);
    std::vector<const double*> coef(nsk);
    std::vector<const int32_t*> q(nsk);
    std::vector<int64_t> width(nsk);
    std::vector<int> tree(nsk);
    std::vector<double*> Up(nsk), Vp(nsk);
    for (int s = 0; s < nsk; ++s) {
      width[s] = std::get<0>(plans[s]);
      tree[s] = std::get<1>(plans[s]);
      src[s] = ptr<const int64_t>(std::get<2>(plans[s]));
      coef[s] = ptr<const double>(std::get<3>(plans[s]));
      q[s] = ptr<const int32_t>(std::get<4>(plans[s]));
      Up[s] = ptr<double>(U[s]);
      Vp[s] = ptr<double>(V[s]);
    }
    std::vector<int32_t> status(nsk, 0);
    check(slra_range_finder_batched(device_context(), ptr<double>(M), ldm, mm, n, nsk, src.data(), coef.data(),
                                    q.data(), width.data(), tree.data(), l, r, truncated ? 1 : 0, Up.data(), ldu,
                                    Vp.data(), ldv, ptr<double>(out), nullptr, status.data()),
          "range_finder_batched");
    for (int s = 0; s < nsk; ++s) check(status[s], "range_finder_batched");
  });
  m.def("cross_approx_batched_device", [](uintptr_t A, Index lda, Index stride, Index nblocks, Index mm, Index n,
                                          Index r, Index k, Index l, uintptr_t init_rows, int loops, double h,
                                          uintptr_t I, uintptr_t J, uintptr_t U, uintptr_t rr, uintptr_t status,
                                          uintptr_t rs, uintptr_t ns) {
    check(slra_cross_approx_batched(device_context(), ptr<double>(A), lda, stride, nblocks, mm, n, r, k, l,
                                    ptr<int64_t>(init_rows), loops, h, ptr<int64_t>(I), ptr<int64_t>(J),
                                    ptr<double>(U), ptr<int64_t>(rr), ptr<int32_t>(status), ptr<double>(rs),
                                    ptr<double>(ns)),
          "cross_approx_batched");
  });
  // §8e multi-GPU over the C-ABI's NCCL communicator (one process per GPU)
  m.def("comm_available", []() { return slra_comm_available() != 0; });
  m.def("comm_unique_id", []() {
    std::string id(SLRA_COMM_ID_BYTES, '\0');
    check(slra_comm_unique_id(id.data()), "comm_unique_id");
    return py::bytes(id);
  });
  m.def("comm_init", [](int nranks, int rank, const py::bytes& id) {
    std::string s = id;
    if (s.size() != SLRA_COMM_ID_BYTES) throw std::invalid_argument("comm_init: id must be 128 bytes");
    slra_comm c = nullptr;
    {
      py::gil_scoped_release nogil;
      check(slra_comm_init(device_context(), nranks, rank, s.data(), &c), "comm_init");
    }
    return reinterpret_cast<uintptr_t>(c);
  });
  m.def("comm_destroy", [](uintptr_t c) { check(slra_comm_destroy(reinterpret_cast<slra_comm>(c)), "comm_destroy"); });
  m.def("comm_allreduce_sum", [](uintptr_t c, uintptr_t send, uintptr_t recv, int64_t count) {
    check(slra_comm_allreduce_sum(reinterpret_cast<slra_comm>(c), ptr<const double>(send), ptr<double>(recv), count),
          "comm_allreduce_sum");
  });
  m.def("comm_allgather", [](uintptr_t c, uintptr_t send, uintptr_t recv, int64_t count) {
    check(slra_comm_allgather(reinterpret_cast<slra_comm>(c), ptr<const double>(send), ptr<double>(recv), count),
          "comm_allgather");
  });
  m.def("sketch_solve_sharded", [](uintptr_t c, uintptr_t A, Index lda, Index m_local, Index d, uintptr_t b,
                                   Index row0, Index m_global, const PyOp& F, bool with_true) {
    LsrReport r = sketch_solve_sharded(reinterpret_cast<slra_comm>(c), ptr<const double>(A), lda, m_local, d,
                                       ptr<const double>(b), row0, m_global, *F.p, with_true);
    py::dict out;
    out["x_hat"] = vec_np(r.x_hat);
    out["sketched_residual"] = r.sketched_residual;
    out["true_residual"] = r.true_residual ? py::cast(*r.true_residual) : py::none();
    out["k"] = r.k;
    return out;
  }, py::arg("comm"), py::arg("A"), py::arg("lda"), py::arg("m_local"), py::arg("d"), py::arg("b"), py::arg("row0"),
     py::arg("m_global"), py::arg("F"), py::arg("with_true_residual") = false);
  // end-to-end batched C-A over HOST blocks (pinned): chunks streamed to the device, results back
  m.def("cross_approx_batched_host", [](uintptr_t A, Index lda, Index stride, Index nblocks, Index mm, Index n,
                                        Index r, Index k, Index l, uintptr_t init_rows, int loops, double h,
                                        uintptr_t I, uintptr_t J, uintptr_t U, uintptr_t rr, uintptr_t status,
                                        uintptr_t rs, uintptr_t ns) {
    py::gil_scoped_release nogil;
    check(slra_cross_approx_batched_host(device_context(), ptr<const double>(A), lda, stride, nblocks, mm, n, r, k,
                                         l, ptr<const int64_t>(init_rows), loops, h, ptr<int64_t>(I),
                                         ptr<int64_t>(J), ptr<double>(U), ptr<int64_t>(rr), ptr<int32_t>(status),
                                         ptr<double>(rs), ptr<double>(ns)),
          "cross_approx_batched_host");
  });
  // config 3's Cauchy block as a FunctionOracle (points on the device)
  m.def("cross_approx_cauchy_device", [](uintptr_t x, uintptr_t y, Index mm, Index n, Index r, Index k, Index l,
                                         uintptr_t init_rows, int loops, double h, uintptr_t I, uintptr_t J,
                                         uintptr_t U, uintptr_t Tsig, uintptr_t Sr) {
    int64_t rr = 0;
    check(slra_cross_approx_cauchy(device_context(), ptr<const double>(x), ptr<const double>(y), mm, n, r, k, l,
                                   ptr<const int64_t>(init_rows), loops, h, ptr<int64_t>(I), ptr<int64_t>(J),
                                   ptr<double>(U), nullptr, nullptr, nullptr, ptr<double>(Tsig), ptr<double>(Sr), &rr),
          "cross_approx_cauchy");
    return rr;
  });
  m.def("cur_residual_factored_cauchy_device", [](uintptr_t x, uintptr_t y, Index mm, Index n, uintptr_t I, Index k,
                                                  uintptr_t J, Index l, uintptr_t Tsig, uintptr_t Sr, Index r,
                                                  uintptr_t out) {
    check(slra_cur_residual_factored_cauchy(device_context(), ptr<const double>(x), ptr<const double>(y), mm, n,
                                            ptr<const int64_t>(I), k, ptr<const int64_t>(J), l,
                                            ptr<const double>(Tsig), ptr<const double>(Sr), r, ptr<double>(out)),
          "cur_residual_factored_cauchy");
  });
  // the same over log-kernel blocks given by their points (FunctionOracle): device / host buffers
  m.def("cross_approx_batched_logkernel_device", [](uintptr_t px, uintptr_t py, uintptr_t qx, uintptr_t qy,
                                                    Index nblocks, Index mm, Index n, Index r, Index k, Index l,
                                                    uintptr_t init_rows, int loops, double h, uintptr_t I,
                                                    uintptr_t J, uintptr_t U, uintptr_t rr, uintptr_t status,
                                                    uintptr_t rs, uintptr_t ns) {
    check(slra_cross_approx_batched_logkernel(device_context(), ptr<const double>(px), ptr<const double>(py),
                                              ptr<const double>(qx), ptr<const double>(qy), nblocks, mm, n, r, k, l,
                                              ptr<const int64_t>(init_rows), loops, h, ptr<int64_t>(I),
                                              ptr<int64_t>(J), ptr<double>(U), ptr<int64_t>(rr),
                                              ptr<int32_t>(status), ptr<double>(rs), ptr<double>(ns)),
          "cross_approx_batched_logkernel");
  });
  m.def("cross_approx_batched_logkernel_host", [](uintptr_t px, uintptr_t py, uintptr_t qx, uintptr_t qy,
                                                  Index nblocks, Index mm, Index n, Index r, Index k, Index l,
                                                  uintptr_t init_rows, int loops, double h, uintptr_t I, uintptr_t J,
                                                  uintptr_t U, uintptr_t rr, uintptr_t status, uintptr_t rs,
                                                  uintptr_t ns) {
    py::gil_scoped_release nogil;
    check(slra_cross_approx_batched_logkernel_host(device_context(), ptr<const double>(px), ptr<const double>(py),
                                                   ptr<const double>(qx), ptr<const double>(qy), nblocks, mm, n, r,
                                                   k, l, ptr<const int64_t>(init_rows), loops, h, ptr<int64_t>(I),
                                                   ptr<int64_t>(J), ptr<double>(U), ptr<int64_t>(rr),
                                                   ptr<int32_t>(status), ptr<double>(rs), ptr<double>(ns)),
          "cross_approx_batched_logkernel_host");
  });
  // config-5 inputs: host points (reference Rng) -> device blocks
  m.def("gen_log_kernel_batch", [](std::uint64_t master, Index b0, Index nb, Index mm, Index n, Index k,
                                   uintptr_t px, uintptr_t py, uintptr_t qx, uintptr_t qy, uintptr_t init) {
    py::gil_scoped_release nogil;
    gen_log_kernel_batch(master, b0, nb, mm, n, k, ptr<double>(px), ptr<double>(py), ptr<double>(qx),
                         ptr<double>(qy), ptr<Index>(init));
  });
  m.def("gen_log_kernel_blocks_device", [](uintptr_t px, uintptr_t py, uintptr_t qx, uintptr_t qy, Index nb,
                                           Index mm, Index n, uintptr_t A, Index lda, Index stride) {
    check(slra_gen_log_kernel_blocks(device_context(), ptr<double>(px), ptr<double>(py), ptr<double>(qx),
                                     ptr<double>(qy), nb, mm, n, ptr<double>(A), lda, stride),
          "gen_log_kernel_blocks");
  });
  m.def("cross_approx_device", [](uintptr_t A, Index lda, Index mm, Index n, Index r, Index k, Index l,
                                  uintptr_t init_rows, int loops, double h, uintptr_t I, uintptr_t J, uintptr_t U,
                                  uintptr_t Tsig, uintptr_t Sr) {
    int64_t r_used = 0;
    check(slra_cross_approx(device_context(), ptr<double>(A), lda, mm, n, r, k, l, ptr<int64_t>(init_rows), loops, h,
                            ptr<int64_t>(I), ptr<int64_t>(J), ptr<double>(U), nullptr, nullptr, nullptr,
                            ptr<double>(Tsig), ptr<double>(Sr), &r_used),
          "cross_approx");
    return r_used;
  }, py::arg("A"), py::arg("lda"), py::arg("m"), py::arg("n"), py::arg("r"), py::arg("k"), py::arg("l"),
     py::arg("init_rows"), py::arg("loops"), py::arg("h"), py::arg("I"), py::arg("J"), py::arg("U"),
     py::arg("Tsig") = 0, py::arg("Sr") = 0);
  m.def("primitive_cur_device", [](uintptr_t A, Index lda, Index mm, Index n, uintptr_t I, Index k, uintptr_t J,
                                   Index l, Index r, uintptr_t U, uintptr_t Tsig, uintptr_t Sr) {
    int64_t r_used = 0;
    check(slra_primitive_cur(device_context(), ptr<double>(A), lda, mm, n, ptr<int64_t>(I), k, ptr<int64_t>(J), l, r,
                             ptr<double>(U), l, ptr<double>(Tsig), ptr<double>(Sr), &r_used),
          "primitive_cur");
    return r_used;
  });
  m.def("cur_residual_factored_device", [](uintptr_t A, Index lda, Index mm, Index n, uintptr_t I, Index k,
                                           uintptr_t J, Index l, uintptr_t Tsig, uintptr_t Sr, Index r,
                                           uintptr_t out) {
    check(slra_cur_residual_factored(device_context(), ptr<double>(A), lda, mm, n, ptr<int64_t>(I), k,
                                     ptr<int64_t>(J), l, ptr<double>(Tsig), ptr<double>(Sr), r, ptr<double>(out)),
          "cur_residual_factored");
  });
  // ---- building blocks of the row-sharded drivers (shard.py)
  m.def("gather_rows_device", [](uintptr_t A, Index lda, Index mm, Index n, uintptr_t I, Index k, uintptr_t R,
                                 Index ldr) {
    check(slra_gather_rows(device_context(), ptr<double>(A), lda, mm, n, ptr<int64_t>(I), k, ptr<double>(R), ldr),
          "gather_rows");
  });
  m.def("gather_cols_device", [](uintptr_t A, Index lda, Index mm, Index n, uintptr_t J, Index l, uintptr_t Cm,
                                 Index ldc) {
    check(slra_gather_cols(device_context(), ptr<double>(A), lda, mm, n, ptr<int64_t>(J), l, ptr<double>(Cm), ldc),
          "gather_cols");
  });
  m.def("select_rows_spanning_device", [](uintptr_t A, Index lda, Index mm, Index c, Index count, double h,
                                          uintptr_t idx, uintptr_t vol) {
    check(slra_select_rows_spanning(device_context(), ptr<double>(A), lda, mm, c, count, h, ptr<int64_t>(idx),
                                    ptr<double>(vol)),
          "select_rows_spanning");
  });
  m.def("sketch_rows_device", [](uintptr_t W, Index ldw, Index mm, Index ncols, uintptr_t src, uintptr_t coef,
                                 uintptr_t q, Index width, int tree, Index k, uintptr_t out, Index ldo) {
    check(slra_sketch_rows(device_context(), ptr<double>(W), ldw, mm, ncols, ptr<int64_t>(src), ptr<double>(coef),
                           ptr<int32_t>(q), width, tree, k, ptr<double>(out), ldo),
          "sketch_rows");
  });
  m.def("sketch_rows_shard_device", [](uintptr_t W, Index ldw, Index row0, Index mloc, Index ncols, uintptr_t src,
                                       uintptr_t coef, Index width, Index k, uintptr_t out, Index ldo,
                                       bool transpose) {
    check(slra_sketch_rows_shard(device_context(), ptr<double>(W), ldw, row0, mloc, ncols, ptr<int64_t>(src),
                                 ptr<double>(coef), width, k, ptr<double>(out), ldo, transpose ? 1 : 0),
          "sketch_rows_shard");
  });
  m.def("lsr_solve_sketched_device",[](uintptr_t FW, Index k, Index d, uintptr_t x) {
    double res = 0;
    check(slra_lsr_solve_sketched(device_context(), ptr<double>(FW), k, k, d, ptr<double>(x), &res),
          "lsr_solve_sketched");
    return res;
  });
  m.def("sketch_solve_device", [](uintptr_t A, Index lda, Index mm, Index d, uintptr_t b, uintptr_t src,
                                  uintptr_t coef, uintptr_t q, Index width, int tree, Index k, uintptr_t x) {
    double res = 0;
    check(slra_sketch_solve(device_context(), ptr<double>(A), lda, mm, d, ptr<double>(b), ptr<int64_t>(src),
                            ptr<double>(coef), ptr<int32_t>(q), width, tree, k, ptr<double>(x), &res),
          "sketch_solve");
    return res;
  });
  m.def("lsr_residual_device", [](uintptr_t A, Index lda, Index mm, Index d, uintptr_t b, uintptr_t x,
                                  uintptr_t out) {
    check(slra_lsr_residual(device_context(), ptr<double>(A), lda, mm, d, ptr<double>(b), ptr<double>(x),
                            ptr<double>(out)),
          "lsr_residual");
  });
  m.def("sketch_solve_batched_device", [](uintptr_t A, Index lda, Index mm, Index d, uintptr_t b,
                                          const std::vector<uintptr_t>& src, const std::vector<uintptr_t>& coef,
                                          const std::vector<uintptr_t>& q, const std::vector<int64_t>& width,
                                          const std::vector<int>& tree, Index k, const std::vector<uintptr_t>& x) {
    const int nsk = (int)src.size();
    if ((int)coef.size() != nsk || (int)q.size() != nsk || (int)width.size() != nsk || (int)tree.size() != nsk ||
        (int)x.size() != nsk)
      throw std::invalid_argument("sketch_solve_batched: list lengths differ");
    std::vector<const int64_t*> ps(nsk);
    std::vector<const double*> pc(nsk);
    std::vector<const int32_t*> pq(nsk);
    std::vector<double*> px(nsk);
    for (int s = 0; s < nsk; ++s) {
      ps[s] = ptr<const int64_t>(src[s]);
      pc[s] = ptr<const double>(coef[s]);
      pq[s] = ptr<const int32_t>(q[s]);
      px[s] = ptr<double>(x[s]);
    }
    std::vector<double> res(nsk, 0.0);
    check(slra_sketch_solve_batched(device_context(), ptr<const double>(A), lda, mm, d, ptr<const double>(b), nsk,
                                    ps.data(), pc.data(), pq.data(), width.data(), tree.data(), k, px.data(),
                                    res.data()),
          "sketch_solve_batched");
    return res;
  });
  m.def("lsr_residual_multi_device", [](uintptr_t A, Index lda, Index mm, Index d, uintptr_t b, uintptr_t X,
                                        Index nx, uintptr_t out) {
    check(slra_lsr_residual_multi(device_context(), ptr<double>(A), lda, mm, d, ptr<double>(b), ptr<double>(X), nx,
                                  ptr<double>(out)),
          "lsr_residual_multi");
  });
  m.def("gemm_device", [](int ta, int tb, Index mm, Index n, Index k, double alpha, uintptr_t A, Index lda,
                          uintptr_t B, Index ldb, double beta, uintptr_t Cm, Index ldc) {
    check(slra_gemm(device_context(), ta, tb, mm, n, k, alpha, ptr<double>(A), lda, ptr<double>(B), ldb, beta,
                    ptr<double>(Cm), ldc),
          "gemm");
  });
  m.def("lowrank_residual_device", [](uintptr_t A, Index lda, Index mm, Index n, uintptr_t P, Index ldp, uintptr_t Q,
                                      Index ldq, Index inner, uintptr_t out) {
    check(slra_lowrank_residual(device_context(), ptr<double>(A), lda, mm, n, ptr<double>(P), ldp, ptr<double>(Q),
                                ldq, inner, ptr<double>(out)),
          "lowrank_residual");
  });
  m.def("cur_residual_device", [](uintptr_t A, Index lda, Index mm, Index n, uintptr_t I, Index k, uintptr_t J,
                                  Index l, uintptr_t U) {
    double rs = 0, ns = 0;
    check(slra_cur_residual(device_context(), ptr<double>(A), lda, mm, n, ptr<int64_t>(I), k, ptr<int64_t>(J), l,
                            ptr<double>(U), l, &rs, &ns),
          "cur_residual");
    return py::make_tuple(rs, ns);
  });
}
