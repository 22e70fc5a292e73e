// CUR / Cross-Approximation entry points of
// /root/reference/proj/include/slra/cur.hpp:16-73, run on the B200.
#pragma once

#include <optional>
#include <utility>
#include <vector>

#include "slra/linalg.hpp"
#include "slra/oracle.hpp"
#include "slra/rng.hpp"

namespace slra {

struct CurDecomposition {
  IndexSet row_set;  // k selected rows
  IndexSet col_set;  // l selected columns
  Matrix nucleus;    // l x k
  Index r = 0;
  bool qr_nucleus = false;  // nucleus from CompleteOrthogonalDecomposition (slra_cod_pinv)
  // Factored nucleus U = tsig * sr^T (l x r, k x r), filled by primitive_cur /
  // cross_approx: cur_evaluate then runs its pass over M at inner dimension r.
  Matrix tsig, sr;
};

/// C * U * R (evaluation only; cur.cpp:76-78).
Matrix cur_reconstruct(const Matrix& M, const CurDecomposition& c);
/// ||M - C U R|| (cur.cpp:80-82). Frobenius runs on the device in one pass
/// over M; Spectral/Chebyshev are not on the hot path (invalid_argument).
double cur_evaluate(const Matrix& M, const CurDecomposition& c, NormKind norm);
double cur_evaluate(const EntryOracle& M, const CurDecomposition& c, NormKind norm);

double t_factor(Index q, Index s, double h);

/// cur.cpp:170-188: maxvol selections inside the top-r factors of a random
/// p x q sub-block, then primitive_cur on M.
CurDecomposition cynical_cur(const EntryOracle& M, Index p, Index q, Index k, Index l, Index r, Rng& rng);
/// cur.cpp:257-272: top-r SVD of A W B through two thin QRs.
Svd lra_to_top_svd(const Matrix& A, const Matrix& W, const Matrix& B, Index r);
enum class CurSelector { Deterministic, Sampled };
/// cur.cpp:278-323: index sets from the singular factors (maxvol or
/// norm-square sampling), nucleus pinv(T_J^T) Sigma^-1 pinv(S_I).
CurDecomposition top_svd_to_cur(const Svd& f, Index k, Index l, double h, CurSelector selector, Rng& rng);
IndexSet maxvol_rows(const Matrix& A, double h = 1.1, Index max_swaps = 0);
IndexSet select_rows_spanning(const Matrix& A, Index count, double h = 1.1);

/// r <= 0 selects the adaptive rank numerical_rank(G, 1e-10, Relative)
/// (configs 3/5); the reference requires r >= 1.
CurDecomposition primitive_cur(const EntryOracle& M, IndexSet I, IndexSet J, Index r,
                               bool qr_nucleus = false);
CurDecomposition primitive_cur(const Matrix& M, IndexSet I, IndexSet J, Index r,
                               bool qr_nucleus = false);

struct CaStep {
  bool horizontal = false;
  std::vector<Index> rows, cols;
  double volume_proxy = 0;
  std::optional<double> error_estimate;
};
struct CaTrace {
  std::vector<CaStep> steps;
};

/// cross_approx (cur.cpp:201-255). The whole loop runs in one CTA-resident
/// kernel; with stop_tol the half-sweeps are host-driven over the device
/// primitives and posterior_error_estimate (lra.cpp:88-127) runs on the device.
std::pair<CurDecomposition, CaTrace> cross_approx(const EntryOracle& M, Index r, Index k, Index l,
                                                  IndexSet init_rows, int loops, double h,
                                                  std::optional<double> stop_tol, Rng& rng);

/// Batched cross_approx + per-block cur_evaluate(M, c, Frobenius) over
/// `nblocks` independent m x n column-major blocks (block b at
/// blocks + b*block_stride, ld = lda) in HOST memory — the per-block
/// ca_factors -> cross_approx pattern of hss.cpp:47-55 applied to a batch.
/// init_rows holds k initial rows per block (nblocks x k); r <= 0 selects the
/// adaptive rank numerical_rank(M(I,J), 1e-10, Relative). The blocks are
/// streamed to the device in chunks (copies overlapped with the kernels);
/// I_out / J_out / nucleus_out (nullable, nblocks x k / x l / x (l*k)) and the
/// returned per-block status, r and squared norms are host data. A block
/// whose selection or generator fails gets its status code (slra_status)
/// and resid_sq = norm_sq instead of an exception, so one bad block does not
/// abort the batch.
struct BatchedCaResult {
  std::vector<int> status;
  std::vector<Index> r;
  std::vector<double> resid_sq, norm_sq;
};
BatchedCaResult cross_approx_batched(const double* blocks, Index lda, Index block_stride, Index nblocks, Index m,
                                     Index n, Index r, Index k, Index l, const Index* init_rows, int loops, double h,
                                     Index* I_out, Index* J_out, double* nucleus_out);

}  // namespace slra
