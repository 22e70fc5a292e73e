// TEST INFRASTRUCTURE ONLY (see slra_oracle.hpp). Restates
// /root/reference/proj/src/linalg.cpp and src/rng.cpp, plus the Eigen
// decompositions they call (HouseholderQR, ColPivHouseholderQR, BDCSVD).
#include <algorithm>
#include <cmath>
#include <limits>
#include <numbers>

#include "slra_oracle.hpp"

namespace slra_oracle {

// ------------------------------------------------------------ Matrix helpers
Matrix Matrix::identity(Index rows, Index cols) {
  Matrix I(rows, cols);
  for (Index i = 0; i < std::min(rows, cols); ++i) I(i, i) = 1.0;
  return I;
}
Matrix Matrix::transpose() const {
  Matrix T(c, r);
  for (Index j = 0; j < c; ++j)
    for (Index i = 0; i < r; ++i) T(j, i) = (*this)(i, j);
  return T;
}
Matrix Matrix::left_cols(Index n) const {
  Matrix out(r, n);
  std::copy(v.begin(), v.begin() + r * n, out.v.begin());
  return out;
}
Matrix Matrix::top_rows(Index n) const {
  Matrix out(n, c);
  for (Index j = 0; j < c; ++j)
    for (Index i = 0; i < n; ++i) out(i, j) = (*this)(i, j);
  return out;
}

// ------------------------------------------------------------ IndexSet
// linalg.cpp:10-29
IndexSet::IndexSet(std::vector<Index> idx, Index bound) : idx_(std::move(idx)), bound_(bound) {
  std::vector<bool> seen(static_cast<size_t>(bound), false);
  for (Index i : idx_) {
    if (i < 0 || i >= bound) throw std::invalid_argument("IndexSet: index out of bound");
    if (seen[static_cast<size_t>(i)]) throw std::invalid_argument("IndexSet: duplicate index");
    seen[static_cast<size_t>(i)] = true;
  }
}
IndexSet IndexSet::iota(Index count, Index bound) {
  std::vector<Index> v(static_cast<size_t>(count));
  for (Index i = 0; i < count; ++i) v[static_cast<size_t>(i)] = i;
  return IndexSet(std::move(v), bound);
}
bool IndexSet::contains(Index i) const {
  for (Index j : idx_)
    if (j == i) return true;
  return false;
}

// ------------------------------------------------------------ Rng
// rng.cpp:8-66 (std::mt19937_64 is specified by the C++ standard).
double Rng::gaussian() {
  double u1 = uniform();
  while (u1 <= 0.0) u1 = uniform();
  const double u2 = uniform();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
}
Index Rng::uniform_index(Index n) {
  const std::uint64_t un = static_cast<std::uint64_t>(n);
  const std::uint64_t limit = UINT64_MAX - UINT64_MAX % un;
  std::uint64_t x = next_u64();
  while (x >= limit) x = next_u64();
  return static_cast<Index>(x % un);
}
std::vector<Index> Rng::permutation(Index n) {
  std::vector<Index> p(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) p[static_cast<size_t>(i)] = i;
  for (Index i = n - 1; i > 0; --i)
    std::swap(p[static_cast<size_t>(i)], p[static_cast<size_t>(uniform_index(i + 1))]);
  return p;
}
std::vector<Index> Rng::distinct_indices(Index k, Index n) {
  std::vector<Index> pool(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) pool[static_cast<size_t>(i)] = i;
  std::vector<Index> out;
  out.reserve(static_cast<size_t>(k));
  for (Index t = 0; t < k; ++t) {
    const Index j = t + uniform_index(n - t);
    std::swap(pool[static_cast<size_t>(t)], pool[static_cast<size_t>(j)]);
    out.push_back(pool[static_cast<size_t>(t)]);
  }
  return out;
}
Matrix Rng::gaussian_matrix(Index rows, Index cols) {
  Matrix G(rows, cols);
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) G(i, j) = gaussian();
  return G;
}
Vector Rng::gaussian_vector(Index n) {
  Vector v(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) v[static_cast<size_t>(i)] = gaussian();
  return v;
}
std::uint64_t Rng::derive_seed(std::uint64_t master, std::uint64_t stream) {
  std::uint64_t z = master + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------ dense products
// Plain column-major products; OpenMP over output columns only, so results
// are bit-identical for every thread count.
Matrix matmul(const Matrix& A, const Matrix& B) {
  if (A.cols() != B.rows()) throw std::invalid_argument("matmul: dimension mismatch");
  const Index m = A.rows(), n = B.cols(), K = A.cols();
  Matrix C(m, n);
#pragma omp parallel for schedule(static)
  for (Index j = 0; j < n; ++j) {
    double* cj = C.col(j);
    for (Index p = 0; p < K; ++p) {
      const double b = B(p, j);
      const double* ap = A.col(p);
      for (Index i = 0; i < m; ++i) cj[i] += ap[i] * b;
    }
  }
  return C;
}
Matrix matmul_tn(const Matrix& A, const Matrix& B) {
  if (A.rows() != B.rows()) throw std::invalid_argument("matmul_tn: dimension mismatch");
  const Index m = A.cols(), n = B.cols(), K = A.rows();
  Matrix C(m, n);
#pragma omp parallel for schedule(static)
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) {
      double s = 0;
      const double* a = A.col(i);
      const double* b = B.col(j);
      for (Index p = 0; p < K; ++p) s += a[p] * b[p];
      C(i, j) = s;
    }
  return C;
}
Matrix sub(const Matrix& A, const Matrix& B) {
  Matrix C(A.rows(), A.cols());
  for (Index t = 0; t < A.size(); ++t) C.v[static_cast<size_t>(t)] = A.v[static_cast<size_t>(t)] - B.v[static_cast<size_t>(t)];
  return C;
}

Matrix select_rows(const Matrix& A, const IndexSet& I) {
  Matrix out(I.size(), A.cols());
  for (Index j = 0; j < A.cols(); ++j)
    for (Index t = 0; t < I.size(); ++t) out(t, j) = A(I[t], j);
  return out;
}
Matrix select_cols(const Matrix& A, const IndexSet& J) {
  Matrix out(A.rows(), J.size());
  for (Index t = 0; t < J.size(); ++t) std::copy(A.col(J[t]), A.col(J[t]) + A.rows(), out.col(t));
  return out;
}
Matrix select_block(const Matrix& A, const IndexSet& I, const IndexSet& J) {
  Matrix out(I.size(), J.size());
  for (Index s = 0; s < I.size(); ++s)
    for (Index t = 0; t < J.size(); ++t) out(s, t) = A(I[s], J[t]);
  return out;
}

// ------------------------------------------------------------ Householder
namespace {

// Eigen MatrixBase::makeHouseholder (Householder.h): x = [c0; tail] ->
// (essential, tau, beta) with H x = beta e0, H = I - tau [1;ess][1;ess]^T.
void make_householder(double* x, Index len, double& tau, double& beta) {
  double tail_sq = 0;
  for (Index i = 1; i < len; ++i) tail_sq += x[i] * x[i];
  const double c0 = x[0];
  const double tol = std::numeric_limits<double>::min();
  if (tail_sq <= tol) {
    tau = 0;
    beta = c0;
    for (Index i = 1; i < len; ++i) x[i] = 0;
  } else {
    beta = std::sqrt(c0 * c0 + tail_sq);
    if (c0 >= 0) beta = -beta;
    const double denom = c0 - beta;
    for (Index i = 1; i < len; ++i) x[i] /= denom;
    tau = (beta - c0) / beta;
  }
}

// Eigen applyHouseholderOnTheLeft: rows [k, k+len) of columns [c0, c1) of X,
// reflector essential part ess[1..len).
void apply_householder_left(Matrix& X, Index k, Index len, const double* ess, double tau, Index c0,
                            Index c1) {
  if (len == 1) {
    for (Index j = c0; j < c1; ++j) X(k, j) *= (1.0 - tau);
    return;
  }
  if (tau == 0) return;
  for (Index j = c0; j < c1; ++j) {
    double* xj = X.col(j) + k;
    double tmp = 0;
    for (Index i = 1; i < len; ++i) tmp += ess[i] * xj[i];
    tmp += xj[0];
    xj[0] -= tau * tmp;
    for (Index i = 1; i < len; ++i) xj[i] -= tau * ess[i] * tmp;
  }
}

struct HouseholderQRResult {
  Matrix qr;
  Vector tau;
};

// Eigen HouseholderQR (unblocked form).
HouseholderQRResult householder_qr(const Matrix& A) {
  HouseholderQRResult out{A, Vector(static_cast<size_t>(std::min(A.rows(), A.cols())))};
  const Index m = A.rows(), n = A.cols(), size = std::min(m, n);
  for (Index k = 0; k < size; ++k) {
    double* x = out.qr.col(k) + k;
    double tau, beta;
    make_householder(x, m - k, tau, beta);
    x[0] = beta;
    out.tau[static_cast<size_t>(k)] = tau;
    apply_householder_left(out.qr, k, m - k, x, tau, k + 1, n);
  }
  return out;
}

// Q * I_thin: apply H_{size-1}, ..., H_0 to the first `cols` unit vectors.
Matrix form_q(const Matrix& qr, const Vector& tau, Index cols) {
  const Index m = qr.rows(), size = static_cast<Index>(tau.size());
  Matrix Q = Matrix::identity(m, cols);
  for (Index k = size - 1; k >= 0; --k) {
    std::vector<double> ess(static_cast<size_t>(m - k));
    ess[0] = 1.0;
    for (Index i = 1; i < m - k; ++i) ess[static_cast<size_t>(i)] = qr(k + i, k);
    apply_householder_left(Q, k, m - k, ess.data(), tau[static_cast<size_t>(k)], 0, cols);
  }
  return Q;
}

}  // namespace

// linalg.cpp:67-79
std::pair<Matrix, Matrix> thin_qr(const Matrix& A) {
  if (A.rows() < A.cols()) throw std::invalid_argument("thin_qr: rows < cols");
  HouseholderQRResult h = householder_qr(A);
  const Index n = A.cols();
  Matrix Q = form_q(h.qr, h.tau, n);
  Matrix R(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i <= j; ++i) R(i, j) = h.qr(i, j);
  for (Index i = 0; i < n; ++i) {
    if (R(i, i) < 0) {
      for (Index j = 0; j < n; ++j) R(i, j) = -R(i, j);
      for (Index t = 0; t < A.rows(); ++t) Q(t, i) = -Q(t, i);
    }
  }
  return {std::move(Q), std::move(R)};
}

// ------------------------------------------------------------ ColPivHouseholderQR
// Eigen ColPivHouseholderQR::computeInPlace (LAPACK xGEQP3 norm downdate).
ColPivQR::ColPivQR(const Matrix& A) : qr(A) {
  const Index rows = A.rows(), cols = A.cols(), size = std::min(rows, cols);
  hcoeffs.assign(static_cast<size_t>(size), 0.0);
  std::vector<Index> transpositions(static_cast<size_t>(size));
  std::vector<double> norms_upd(static_cast<size_t>(cols)), norms_dir(static_cast<size_t>(cols));
  for (Index k = 0; k < cols; ++k) {
    double s = 0;
    for (Index i = 0; i < rows; ++i) s += qr(i, k) * qr(i, k);
    norms_upd[static_cast<size_t>(k)] = norms_dir[static_cast<size_t>(k)] = std::sqrt(s);
  }
  double maxnorm = 0;
  for (double v : norms_upd) maxnorm = std::max(maxnorm, v);
  const double eps = std::numeric_limits<double>::epsilon();
  const double threshold_helper = (maxnorm * eps) * (maxnorm * eps) / static_cast<double>(rows);
  const double norm_downdate_threshold = std::sqrt(eps);
  nonzero_pivots = size;
  maxpivot = 0;
  for (Index k = 0; k < size; ++k) {
    // maxCoeff(&idx) over the remaining norms: first maximum wins.
    Index big = k;
    double bigv = norms_upd[static_cast<size_t>(k)];
    for (Index j = k + 1; j < cols; ++j)
      if (norms_upd[static_cast<size_t>(j)] > bigv) {
        bigv = norms_upd[static_cast<size_t>(j)];
        big = j;
      }
    const double big_sq = bigv * bigv;
    if (nonzero_pivots == size && big_sq < threshold_helper * static_cast<double>(rows - k))
      nonzero_pivots = k;
    transpositions[static_cast<size_t>(k)] = big;
    if (k != big) {
      for (Index i = 0; i < rows; ++i) std::swap(qr(i, k), qr(i, big));
      std::swap(norms_upd[static_cast<size_t>(k)], norms_upd[static_cast<size_t>(big)]);
      std::swap(norms_dir[static_cast<size_t>(k)], norms_dir[static_cast<size_t>(big)]);
    }
    double tau, beta;
    double* x = qr.col(k) + k;
    make_householder(x, rows - k, tau, beta);
    x[0] = beta;
    hcoeffs[static_cast<size_t>(k)] = tau;
    if (std::abs(beta) > maxpivot) maxpivot = std::abs(beta);
    apply_householder_left(qr, k, rows - k, x, tau, k + 1, cols);
    for (Index j = k + 1; j < cols; ++j) {
      double& nu = norms_upd[static_cast<size_t>(j)];
      double& nd = norms_dir[static_cast<size_t>(j)];
      if (nu != 0) {
        double temp = std::abs(qr(k, j)) / nu;
        temp = (1.0 + temp) * (1.0 - temp);
        temp = temp < 0 ? 0 : temp;
        const double ratio = nu / nd;
        const double temp2 = temp * ratio * ratio;
        if (temp2 <= norm_downdate_threshold) {
          double s = 0;
          for (Index i = k + 1; i < rows; ++i) s += qr(i, j) * qr(i, j);
          nd = std::sqrt(s);
          nu = nd;
        } else {
          nu *= std::sqrt(temp);
        }
      }
    }
  }
  perm.resize(static_cast<size_t>(cols));
  for (Index i = 0; i < cols; ++i) perm[static_cast<size_t>(i)] = i;
  for (Index k = 0; k < size; ++k)
    std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(transpositions[static_cast<size_t>(k)])]);
}

Index ColPivQR::rank() const {
  const double thr = threshold >= 0 ? threshold
                                    : std::numeric_limits<double>::epsilon() *
                                          static_cast<double>(std::min(qr.rows(), qr.cols()));
  const double pre = std::abs(maxpivot) * thr;
  Index result = 0;
  for (Index i = 0; i < nonzero_pivots; ++i) result += (std::abs(qr(i, i)) > pre);
  return result;
}

Matrix ColPivQR::solve(const Matrix& B) const {
  const Index rows = qr.rows(), cols = qr.cols(), np = nonzero_pivots;
  Matrix dst(cols, B.cols());
  if (np == 0) return dst;
  Matrix c = B;
  // c <- H_{np-1} ... H_0 c  (householderQ().setLength(np).adjoint())
  for (Index k = 0; k < np; ++k)
    apply_householder_left(c, k, rows - k, qr.col(k) + k, hcoeffs[static_cast<size_t>(k)], 0, c.cols());
  // note: apply_householder_left reads ess[1..len) = qr(k+1.., k); ess[0] unused.
  for (Index j = 0; j < c.cols(); ++j) {
    for (Index i = np - 1; i >= 0; --i) {
      double s = c(i, j);
      for (Index t = i + 1; t < np; ++t) s -= qr(i, t) * c(t, j);
      c(i, j) = s / qr(i, i);
    }
  }
  for (Index i = 0; i < np; ++i)
    for (Index j = 0; j < c.cols(); ++j) dst(perm[static_cast<size_t>(i)], j) = c(i, j);
  return dst;
}

// ------------------------------------------------------------ CompleteOrthogonalDecomposition
// Eigen CompleteOrthogonalDecomposition as primitive_cur's qr_nucleus branch
// uses it (cur.cpp:146-152): `cod(G)` factors G at construction, so the
// RZ step (computeInPlace) runs at the DEFAULT ColPivQR rank (threshold
// eps * min(k, l)); `setThreshold(1e-10)` then changes rank(), which both the
// caller's check and pseudoInverse() (_solve_impl with an identity rhs) read.
// Restated step by step, including that ordering: the RZ reflectors are
// built for the default rank r_e, applied (applyZAdjointOnTheLeftInPlace)
// with the thresholded rank r_t. Where Eigen reads z-coefficients it never
// wrote (r_e == l > r_t: m_zCoeffs is resized, not set) tau = 0 is used.
Matrix cod_pseudo_inverse(const Matrix& G, double threshold, Index* rank_out) {
  const Index rows = G.rows(), cols = G.cols();
  ColPivQR cp(G);
  Matrix& X = cp.qr;
  const Index r_e = cp.rank();  // default threshold: the rank computeInPlace sees
  std::vector<double> zc(static_cast<size_t>(std::min(rows, cols)), 0.0);
  if (r_e < cols) {
    // [R11 R12] = [T11 0] Z, Householder from the right, last row first
    for (Index k = r_e - 1; k >= 0; --k) {
      if (k != r_e - 1)
        for (Index i = 0; i <= k; ++i) std::swap(X(i, k), X(i, r_e - 1));
      // row(k).tail(cols - r_e + 1), starting at column r_e - 1
      const Index len = cols - r_e + 1;
      std::vector<double> x(static_cast<size_t>(len));
      for (Index j = 0; j < len; ++j) x[static_cast<size_t>(j)] = X(k, r_e - 1 + j);
      double tau, beta;
      make_householder(x.data(), len, tau, beta);
      for (Index j = 1; j < len; ++j) X(k, r_e - 1 + j) = x[static_cast<size_t>(j)];
      zc[static_cast<size_t>(k)] = tau;
      X(k, r_e - 1) = beta;
      // applyHouseholderOnTheRight on topRightCorner(k, len), essential = row k tail
      if (k > 0 && tau != 0) {
        for (Index i = 0; i < k; ++i) {
          double tmp = 0;
          for (Index j = 1; j < len; ++j) tmp += X(i, r_e - 1 + j) * x[static_cast<size_t>(j)];
          tmp += X(i, r_e - 1);
          X(i, r_e - 1) -= tau * tmp;
          for (Index j = 1; j < len; ++j) X(i, r_e - 1 + j) -= tau * tmp * x[static_cast<size_t>(j)];
        }
      }
      if (k != r_e - 1)
        for (Index i = 0; i <= k; ++i) std::swap(X(i, k), X(i, r_e - 1));
    }
  }
  cp.threshold = threshold;  // cod.setThreshold(threshold)
  const Index rank = cp.rank();
  if (rank_out) *rank_out = rank;
  Matrix dst(cols, rows);
  if (rank == 0) return dst;
  // c = Q^T I with the first `rank` reflectors (matrixQ().setLength(rank))
  Matrix c = Matrix::identity(rows, rows);
  for (Index k = 0; k < rank; ++k)
    apply_householder_left(c, k, rows - k, X.col(k) + k, cp.hcoeffs[static_cast<size_t>(k)], 0, rows);
  // T11 z = c(0:rank, :)
  for (Index j = 0; j < rows; ++j)
    for (Index i = rank - 1; i >= 0; --i) {
      double s = c(i, j);
      for (Index t = i + 1; t < rank; ++t) s -= X(i, t) * dst(t, j);
      dst(i, j) = s / X(i, i);
    }
  if (rank < cols) {
    // applyZAdjointOnTheLeftInPlace(dst), essential = row k, columns rank..cols-1
    const Index len = cols - rank + 1;
    std::vector<double> ess(static_cast<size_t>(len));
    for (Index k = 0; k < rank; ++k) {  // Z^T = Z(r-1) ... Z(0): Z(0) first
      if (k != rank - 1)
        for (Index j = 0; j < rows; ++j) std::swap(dst(k, j), dst(rank - 1, j));
      ess[0] = 1.0;
      for (Index j = 1; j < len; ++j) ess[static_cast<size_t>(j)] = X(k, rank - 1 + j);
      apply_householder_left(dst, rank - 1, len, ess.data(), zc[static_cast<size_t>(k)], 0, rows);
      if (k != rank - 1)
        for (Index j = 0; j < rows; ++j) std::swap(dst(k, j), dst(rank - 1, j));
    }
  }
  // x = P y
  Matrix out(cols, rows);
  for (Index i = 0; i < cols; ++i)
    for (Index j = 0; j < rows; ++j) out(cp.perm[static_cast<size_t>(i)], j) = dst(i, j);
  return out;
}

// ------------------------------------------------------------ SVD
namespace {

// One-sided (Hestenes) Jacobi on a square W (n x n); accumulates V.
void jacobi_sweeps(Matrix& W, Matrix& V) {
  const Index m = W.rows(), n = W.cols();
  const double eps = std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (Index p = 0; p < n - 1; ++p)
      for (Index q = p + 1; q < n; ++q) {
        double* wp = W.col(p);
        double* wq = W.col(q);
        double a = 0, b = 0, g = 0;
        for (Index i = 0; i < m; ++i) {
          a += wp[i] * wp[i];
          b += wq[i] * wq[i];
          g += wp[i] * wq[i];
        }
        if (g == 0 || std::abs(g) <= eps * std::sqrt(a * b)) continue;
        rotated = true;
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (Index i = 0; i < m; ++i) {
          const double x = wp[i], y = wq[i];
          wp[i] = cs * x - sn * y;
          wq[i] = sn * x + cs * y;
        }
        double* vp = V.col(p);
        double* vq = V.col(q);
        for (Index i = 0; i < V.rows(); ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = cs * x - sn * y;
          vq[i] = sn * x + cs * y;
        }
      }
    if (!rotated) break;
  }
}

// Orthonormal completion for columns whose singular value is exactly zero.
void complete_column(Matrix& S, Index j) {
  const Index m = S.rows();
  for (Index e = 0; e < m; ++e) {
    std::vector<double> u(static_cast<size_t>(m), 0.0);
    u[static_cast<size_t>(e)] = 1.0;
    for (int pass = 0; pass < 2; ++pass)
      for (Index t = 0; t < S.cols(); ++t) {
        if (t == j) continue;
        double d = 0;
        for (Index i = 0; i < m; ++i) d += S(i, t) * u[static_cast<size_t>(i)];
        for (Index i = 0; i < m; ++i) u[static_cast<size_t>(i)] -= d * S(i, t);
      }
    double nrm = 0;
    for (double x : u) nrm += x * x;
    nrm = std::sqrt(nrm);
    if (nrm > 0.5) {
      for (Index i = 0; i < m; ++i) S(i, j) = u[static_cast<size_t>(i)] / nrm;
      return;
    }
  }
}

Svd svd_tall(const Matrix& A) {
  const Index m = A.rows(), n = A.cols();
  Svd out;
  if (n == 0) {
    out.S = Matrix(m, 0);
    out.T = Matrix(0, 0);
    return out;
  }
  // QR pre-reduction, then Jacobi on the n x n triangle.
  HouseholderQRResult h = householder_qr(A);
  Matrix R(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i <= j; ++i) R(i, j) = h.qr(i, j);
  Matrix V = Matrix::identity(n, n);
  jacobi_sweeps(R, V);
  std::vector<double> sig(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) {
    double s = 0;
    for (Index i = 0; i < n; ++i) s += R(i, j) * R(i, j);
    sig[static_cast<size_t>(j)] = std::sqrt(s);
  }
  std::vector<Index> order(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) order[static_cast<size_t>(j)] = j;
  std::stable_sort(order.begin(), order.end(), [&](Index a, Index b) {
    return sig[static_cast<size_t>(a)] > sig[static_cast<size_t>(b)];
  });
  Matrix UR(n, n);
  out.sigma.resize(static_cast<size_t>(n));
  out.T = Matrix(n, n);
  std::vector<bool> zero(static_cast<size_t>(n), false);
  for (Index t = 0; t < n; ++t) {
    const Index j = order[static_cast<size_t>(t)];
    const double s = sig[static_cast<size_t>(j)];
    out.sigma[static_cast<size_t>(t)] = s;
    for (Index i = 0; i < n; ++i) out.T(i, t) = V(i, j);
    if (s > 0)
      for (Index i = 0; i < n; ++i) UR(i, t) = R(i, j) / s;
    else
      zero[static_cast<size_t>(t)] = true;
  }
  for (Index t = 0; t < n; ++t)
    if (zero[static_cast<size_t>(t)]) complete_column(UR, t);
  // S = Q [UR; 0]
  Matrix Ufull(m, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) Ufull(i, j) = UR(i, j);
  for (Index k = std::min(m, n) - 1; k >= 0; --k) {
    std::vector<double> ess(static_cast<size_t>(m - k));
    ess[0] = 1.0;
    for (Index i = 1; i < m - k; ++i) ess[static_cast<size_t>(i)] = h.qr(k + i, k);
    apply_householder_left(Ufull, k, m - k, ess.data(), h.tau[static_cast<size_t>(k)], 0, n);
  }
  out.S = std::move(Ufull);
  return out;
}

}  // namespace

// linalg.cpp:81-98 (BDCSVD replaced by QR + one-sided Jacobi; same sign rule)
Svd svd(const Matrix& A) {
  Svd out;
  if (A.rows() >= A.cols()) {
    out = svd_tall(A);
  } else {
    Svd t = svd_tall(A.transpose());
    out.S = std::move(t.T);
    out.sigma = std::move(t.sigma);
    out.T = std::move(t.S);
  }
  for (Index j = 0; j < out.S.cols(); ++j) {
    Index imax = 0;
    double best = -1;
    for (Index i = 0; i < out.S.rows(); ++i)
      if (std::abs(out.S(i, j)) > best) {
        best = std::abs(out.S(i, j));
        imax = i;
      }
    if (out.S(imax, j) < 0) {
      for (Index i = 0; i < out.S.rows(); ++i) out.S(i, j) = -out.S(i, j);
      for (Index i = 0; i < out.T.rows(); ++i) out.T(i, j) = -out.T(i, j);
    }
  }
  return out;
}

// linalg.cpp:100-109
LowRankFactors truncate_rank(const Matrix& A, Index rho) {
  if (rho < 1 || rho > std::min(A.rows(), A.cols()))
    throw std::invalid_argument("truncate_rank: rho out of range");
  const Svd f = svd(A);
  LowRankFactors out;
  out.U = Matrix(A.rows(), rho);
  for (Index j = 0; j < rho; ++j)
    for (Index i = 0; i < A.rows(); ++i) out.U(i, j) = f.S(i, j) * f.sigma[static_cast<size_t>(j)];
  out.V = f.T.left_cols(rho).transpose();
  out.target_rank = rho;
  return out;
}

// linalg.cpp:111-121
Matrix pseudo_inverse(const Matrix& A, double rank_tol) {
  const Svd f = svd(A);
  if (f.sigma.empty() || f.sigma[0] == 0.0) return Matrix(A.cols(), A.rows());
  const double cut = rank_tol * f.sigma[0];
  Index rho = 0;
  while (rho < static_cast<Index>(f.sigma.size()) && f.sigma[static_cast<size_t>(rho)] > cut) ++rho;
  if (rho == 0) return Matrix(A.cols(), A.rows());
  // T_rho diag(1/sigma) S_rho^T
  Matrix TS(A.cols(), rho);
  for (Index j = 0; j < rho; ++j) {
    const double inv = 1.0 / f.sigma[static_cast<size_t>(j)];
    for (Index i = 0; i < A.cols(); ++i) TS(i, j) = f.T(i, j) * inv;
  }
  Matrix St(rho, A.rows());
  for (Index i = 0; i < A.rows(); ++i)
    for (Index j = 0; j < rho; ++j) St(j, i) = f.S(i, j);
  return matmul(TS, St);
}

// linalg.cpp:123-132
Index numerical_rank(const Matrix& A, double tol, RankMode mode) {
  if (tol <= 0) throw std::invalid_argument("numerical_rank: tol must be positive");
  const Svd f = svd(A);
  if (f.sigma.empty()) return 0;
  const double cut = (mode == RankMode::Absolute) ? tol : tol * f.sigma[0];
  Index count = 0;
  for (double s : f.sigma)
    if (s > cut) ++count;
  return count;
}

double spectral_norm(const Matrix& A) {
  if (A.size() == 0) return 0.0;
  return svd(A).sigma[0];
}
double frobenius_norm(const Matrix& A) {
  double s = 0;
  for (double x : A.v) s += x * x;
  return std::sqrt(s);
}
double chebyshev_norm(const Matrix& A) {
  double m = 0;
  for (double x : A.v) m = std::max(m, std::abs(x));
  return m;
}
double matrix_norm(const Matrix& A, NormKind kind) {
  switch (kind) {
    case NormKind::Spectral: return spectral_norm(A);
    case NormKind::Frobenius: return frobenius_norm(A);
    default: return chebyshev_norm(A);
  }
}

// |det| via partial-pivot LU (Eigen PartialPivLU::determinant).
double determinant_abs(const Matrix& A) {
  const Index n = A.rows();
  Matrix L = A;
  double det = 1.0;
  for (Index k = 0; k < n; ++k) {
    Index p = k;
    for (Index i = k + 1; i < n; ++i)
      if (std::abs(L(i, k)) > std::abs(L(p, k))) p = i;
    if (L(p, k) == 0) return 0.0;
    if (p != k)
      for (Index j = 0; j < n; ++j) std::swap(L(k, j), L(p, j));
    det *= L(k, k);
    for (Index i = k + 1; i < n; ++i) {
      const double f = L(i, k) / L(k, k);
      for (Index j = k + 1; j < n; ++j) L(i, j) -= f * L(k, j);
    }
  }
  return std::abs(det);
}

}  // namespace slra_oracle
