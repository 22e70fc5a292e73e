// Seeded synthetic inputs: same draw order and arithmetic order as
// /root/reference/proj/src/testgen.cpp:110-115, 159-193 (no FMA contraction,
// products accumulated in index order), so the oracle restatement produces
// bit-identical matrices. Input generation is untimed setup, not the path.
#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "slra/testgen.hpp"

namespace slra {

namespace {
// C = A * B accumulated column by column in p order (oracle/src/linalg.cpp matmul)
Matrix host_product(const Matrix& A, const Matrix& B) {
  Matrix C(A.rows(), B.cols());
  for (Index j = 0; j < B.cols(); ++j)
    for (Index p = 0; p < A.cols(); ++p) {
      const double b = B(p, j);
      for (Index i = 0; i < A.rows(); ++i) C(i, j) += A(i, p) * b;
    }
  return C;
}
}  // namespace

Matrix gen_factor_gaussian(Index m, Index n, Index r, double noise, Rng& rng) {
  if (r > std::min(m, n)) throw std::invalid_argument("gen_factor_gaussian: r too large");
  Matrix G1 = rng.gaussian_matrix(m, r);
  Matrix G2 = rng.gaussian_matrix(r, n);
  Matrix M = host_product(G1, G2);
  if (noise != 0) {
    Matrix N = rng.gaussian_matrix(m, n);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) M(i, j) += noise * N(i, j);
  }
  return M;
}

LsrProblem gen_lsr_gaussian(Index m, Index n, double noise, Rng& rng) {
  if (m <= n) throw std::invalid_argument("gen_lsr_family: need m > n");
  LsrProblem p;
  p.A = rng.gaussian_matrix(m, n);
  Vector x0 = rng.gaussian_vector(n);
  Vector e = rng.gaussian_vector(m);
  Matrix X(n, 1);
  for (Index i = 0; i < n; ++i) X(i, 0) = x0[static_cast<size_t>(i)];
  Matrix Ax = host_product(p.A, X);
  p.b.resize(static_cast<size_t>(m));
  for (Index i = 0; i < m; ++i) p.b[static_cast<size_t>(i)] = Ax(i, 0) + noise * e[static_cast<size_t>(i)];
  return p;
}

Matrix gen_cauchy_block(Index m, Index n, Rng& rng) {
  Vector x(static_cast<size_t>(m)), y(static_cast<size_t>(n));
  for (auto& v : x) v = rng.uniform();
  for (auto& v : y) v = 2.0 + rng.uniform();
  Matrix A(m, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) A(i, j) = 1.0 / (x[static_cast<size_t>(i)] - y[static_cast<size_t>(j)]);
  return A;
}

Matrix gen_log_kernel_block(Index m, Index n, Rng& rng) {
  Vector px(static_cast<size_t>(m)), py(static_cast<size_t>(m)), qx(static_cast<size_t>(n)), qy(static_cast<size_t>(n));
  for (Index i = 0; i < m; ++i) {
    px[static_cast<size_t>(i)] = rng.uniform();
    py[static_cast<size_t>(i)] = rng.uniform();
  }
  for (Index j = 0; j < n; ++j) {
    qx[static_cast<size_t>(j)] = 4.0 + rng.uniform();
    qy[static_cast<size_t>(j)] = rng.uniform();
  }
  Matrix K(m, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) {
      const double dx = px[static_cast<size_t>(i)] - qx[static_cast<size_t>(j)];
      const double dy = py[static_cast<size_t>(i)] - qy[static_cast<size_t>(j)];
      K(i, j) = 0.5 * std::log(dx * dx + dy * dy);
    }
  return K;
}

void gen_log_kernel_batch(std::uint64_t master, Index b0, Index nb, Index m, Index n, Index k, double* px,
                          double* py, double* qx, double* qy, Index* init) {
  if (k > m) throw std::invalid_argument("gen_log_kernel_batch: k > m");
  for (Index t = 0; t < nb; ++t) {
    Rng rng(Rng::derive_seed(master, static_cast<std::uint64_t>(b0 + t)));
    for (Index i = 0; i < m; ++i) {
      px[t * m + i] = rng.uniform();
      py[t * m + i] = rng.uniform();
    }
    for (Index j = 0; j < n; ++j) {
      qx[t * n + j] = 4.0 + rng.uniform();
      qy[t * n + j] = rng.uniform();
    }
    const std::vector<Index> ini = rng.distinct_indices(k, m);
    for (Index u = 0; u < k; ++u) init[t * k + u] = ini[static_cast<size_t>(u)];
  }
}

}  // namespace slra

// ------------------------------------------------ bidiagonal-product generator
// sketch.cpp:695-791 (host: input generation and a statistical check)
namespace slra {

Matrix bidiagonal_factor(Index n, const std::vector<int>& signs) {
  if (static_cast<Index>(signs.size()) != n) throw std::invalid_argument("bidiagonal_factor: need n signs");
  Matrix B = Matrix::Identity(n, n);
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

KsResult ks_normality(const std::vector<double>& sample) {
  if (sample.size() < 30) throw std::invalid_argument("ks_normality: need at least 30 samples");
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
  KsResult out;
  out.statistic = d;
  out.pass = d < 1.36 / std::sqrt(static_cast<double>(n));
  return out;
}

}  // namespace slra
