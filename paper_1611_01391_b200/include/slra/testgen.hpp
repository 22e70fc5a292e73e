// Seeded synthetic inputs (/root/reference/proj/include/slra/testgen.hpp), the
// same draw order as the reference generators so the oracle and the device
// path see identical matrices.
#pragma once

#include "slra/lsr.hpp"
#include "slra/rng.hpp"

namespace slra {

/// G1 * G2 + noise * G3 (testgen.cpp:110-115): G1 drawn first, then G2, then G3.
Matrix gen_factor_gaussian(Index m, Index n, Index r, double noise, Rng& rng);
/// Gaussian LSR family (testgen.cpp:159-193) with the noise scale a parameter.
LsrProblem gen_lsr_gaussian(Index m, Index n, double noise, Rng& rng);
/// Config 3: x_i ~ U[0,1] (m draws) then y_j ~ U[2,3] (n draws); A_ij = 1/(x_i - y_j).
Matrix gen_cauchy_block(Index m, Index n, Rng& rng);
/// Config 5 block: p_i = (u,u) in [0,1]^2 (m points), then q_j = (u+4, u);
/// K_ij = 0.5 log((dx)^2 + (dy)^2) = log|p_i - q_j|.
Matrix gen_log_kernel_block(Index m, Index n, Rng& rng);
/// Config-5 batch recipe: block b = b0 + t draws from
/// Rng(derive_seed(master, b)) its points p_i = (u, u) (m), then q_j =
/// (4 + u, u) (n) — gen_log_kernel_block's order — and then its initial C-A
/// rows distinct_indices(k, m) (what cross_approx draws for an empty initial
/// set, cur.cpp:207-209). Arrays are nb x m / nb x n / nb x k, row t = block t.
void gen_log_kernel_batch(std::uint64_t master, Index b0, Index nb, Index m, Index n, Index k, double* px,
                          double* py, double* qx, double* qy, Index* init);

/// Bidiagonal-product pseudo-Gaussian generator (sketch.hpp:92-112,
/// sketch.cpp:695-791): host generators and the KS normality check, drawing
/// in the reference's order.
Matrix bidiagonal_factor(Index n, const std::vector<int>& signs);
Matrix gen_bidiagonal_product(Index n, Index T, Rng& rng, bool standardize = true);
Vector bidiagonal_product_column(Index n, Index T, Index j, Rng& rng);
struct KsResult {
  double statistic = 0;
  bool pass = false;
};
KsResult ks_normality(const std::vector<double>& sample);

}  // namespace slra
