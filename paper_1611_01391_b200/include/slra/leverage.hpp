// Leverage-score sampling and CUR (/root/reference/proj/include/slra/leverage.hpp)
// on the B200: SVDs, gathers, rescaling and pseudo-inverses run on the
// device; the categorical / Bernoulli draws stay on the host Rng (the same
// stream as the reference).
#pragma once

#include <optional>
#include <vector>

#include "slra/cur.hpp"
#include "slra/linalg.hpp"
#include "slra/oracle.hpp"
#include "slra/rng.hpp"

namespace slra {

struct LeverageScores {
  Vector p;
  double beta = 1.0;
  Index r = 0;
};

struct SampleRescale {
  std::vector<Index> indices;
  Vector d;
};

enum class SampleMode { Exactly, Expected };

LeverageScores svd_leverage_scores(const Matrix& T_r, double beta = 1.0);
SampleRescale sample_exactly(const LeverageScores& scores, Index l, Rng& rng);
SampleRescale sample_expected(const LeverageScores& scores, Index l, Rng& rng);
SampleRescale collapse_duplicates(const SampleRescale& s);

CurDecomposition cur_via_leverage(const EntryOracle& M, Index r, Index k, Index l, double beta, double beta_bar,
                                  SampleMode mode, const std::optional<LeverageScores>& scores, Rng& rng,
                                  bool plain_nucleus = false);

/// Top-r SVD of U V through two thin QRs and the SVD of R_U R_V^T (cur.cpp:257-276).
Svd lra_to_top_svd(const LowRankFactors& f, Index r);
CurDecomposition refine_lra(const EntryOracle& M, const LowRankFactors& crude, Index r, Index k, Index l, Rng& rng);

LeverageScores uniform_scores(Index n);
double gaussian_score_gap(const Matrix& G);
double sample_bound_quadratic(Index r, double eps, double beta);
double sample_bound_loglinear(Index r, double eps, double beta, double cbar);
double epsilon_for_sample(Index r, Index l, double delta);

}  // namespace slra
