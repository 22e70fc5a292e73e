// Seeded synthetic inputs: same draw order and arithmetic order as
// /root/reference/proj/src/testgen.cpp:110-115, 159-193 (no FMA contraction,
// products accumulated in index order), so the oracle restatement produces
// bit-identical matrices. Input generation is untimed setup, not the path.
#include <cmath>

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

}  // namespace slra
