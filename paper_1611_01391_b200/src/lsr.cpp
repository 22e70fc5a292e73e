// Sketch-and-solve LSR host entry points (/root/reference/proj/src/lsr.cpp:21-67).
#include <cmath>
#include <limits>

#include "slra/devbuf.hpp"
#include "slra/errors.hpp"
#include "slra/lsr.hpp"

namespace slra {

namespace {
void validate(const LsrProblem& p) {  // lsr.cpp:13-17
  if (p.A.rows() <= p.A.cols() || p.A.cols() < 1) throw std::invalid_argument("lsr: need m > d >= 1");
  if (static_cast<Index>(p.b.size()) != p.A.rows()) throw std::invalid_argument("lsr: b length mismatch");
}

// sketch_solve on an HBM-resident (A, b): one plan, one C-ABI call.
LsrReport sketch_solve_resident(const DeviceMatrix& dA, const double* db, const SketchOperator& F) {
  const Index d = dA.cols(), m = dA.rows();
  if (F.cols() != m) throw std::invalid_argument("sketch_solve: F cols != m");
  if (F.rows() <= d) throw std::invalid_argument("sketch_solve: need k > d");
  if (!F.plannable()) {
    // F holds a non-plan factor (inverse bidiagonal, Householder chain): the
    // sketched system F (A | b) is formed by F's device application into the
    // two column blocks of FW, then solved as the row-sharded path does
    const Index k = F.rows();
    DeviceMatrix FW(k, d + 1);
    DeviceMatrix FA = DeviceMatrix::view(FW.data(), k, d, FW.ld());
    DeviceMatrix Fb = DeviceMatrix::view(FW.data() + FW.ld() * d, k, 1, FW.ld());
    const DeviceMatrix bv = DeviceMatrix::view(const_cast<double*>(db), m, 1, m);
    F.apply_device(dA, false, FA);
    F.apply_device(bv, false, Fb);
    DevBuf<double> dx(static_cast<size_t>(d));
    LsrReport rep;
    check(slra_lsr_solve_sketched(device_context(), FW.data(), FW.ld(), k, d, dx.get(), &rep.sketched_residual),
          "sketch_solve");
    rep.x_hat = dx.download();
    rep.k = k;
    return rep;
  }
  const SketchPlan plan = compile_plan(F, Side::Left);
  DevBuf<double> dx(static_cast<size_t>(d));
  DevBuf<int64_t> src(plan.src);
  DevBuf<double> coef(plan.coef);
  DevBuf<int32_t> q(plan.q);
  LsrReport rep;
  check(slra_sketch_solve(device_context(), dA.data(), dA.ld(), m, d, db, src.get(), coef.get(), q.get(), plan.width,
                          plan.tree, plan.count, dx.get(), &rep.sketched_residual),
        "sketch_solve");
  rep.x_hat = dx.download();
  rep.k = F.rows();
  return rep;
}
}  // namespace

// lsr.cpp:69-113: retries re-randomise the sketch as F Q (Q a fresh random
// permutation, or the caller's family in turn); every solution is validated
// against an independently drawn F P: ||(F P A) x_hat - F P b|| versus the
// sketched residual. (A, b) stay in HBM across attempts; each validation is
// a plan gather of the k sketched rows plus one device residual pass.
LsrReport solve_with_retries(const LsrProblem& p, OpPtr base_F, const std::vector<OpPtr>& q_family,
                             int max_retries, double accept_tol, Rng& rng) {
  validate(p);
  const Index m = p.A.rows(), d = p.A.cols();
  slra_ctx cx = device_context();
  DeviceMatrix dA = DeviceMatrix::upload(p.A);
  DevBuf<double> db(p.b);
  LsrReport best;
  double best_score = std::numeric_limits<double>::infinity();
  bool have_best = false;
  for (int attempt = 0; attempt <= max_retries; ++attempt) {
    OpPtr F = base_F;
    if (attempt > 0) {
      OpPtr Q = q_family.empty() ? gen_permutation(m, rng)
                                 : q_family[static_cast<size_t>((attempt - 1) % static_cast<int>(q_family.size()))];
      F = make_product({base_F, Q});
    }
    LsrReport rep;
    try {
      rep = sketch_solve_resident(dA, db.get(), *F);
    } catch (const SketchRankFailure&) {
      continue;
    }
    rep.attempts = attempt + 1;
    OpPtr Fv = make_product({base_F, gen_permutation(m, rng)});
    const SketchPlan pv = compile_plan(*Fv, Side::Left);
    const Index k = pv.count;
    DevBuf<int64_t> src(pv.src);
    DevBuf<double> coef(pv.coef);
    DevBuf<int32_t> q(pv.q);
    DevBuf<double> VA(static_cast<size_t>(k * d)), vb(static_cast<size_t>(k)), x(rep.x_hat), out(2), zero(
        std::vector<double>(static_cast<size_t>(d), 0.0));
    check(slra_sketch_rows(cx, dA.data(), dA.ld(), m, d, src.get(), coef.get(), q.get(), pv.width, pv.tree, k,
                           VA.get(), k),
          "solve_with_retries");
    check(slra_sketch_rows(cx, db.get(), m, m, 1, src.get(), coef.get(), q.get(), pv.width, pv.tree, k, vb.get(), k),
          "solve_with_retries");
    check(slra_lsr_residual(cx, VA.get(), k, k, d, vb.get(), x.get(), out.get()), "solve_with_retries");
    const double r_val = std::sqrt(out.download()[0]);
    check(slra_lsr_residual(cx, VA.get(), k, k, d, vb.get(), zero.get(), out.get()), "solve_with_retries");
    const double vb_norm = std::sqrt(out.download()[0]);
    const double score = r_val / std::max(rep.sketched_residual, 1e-300);
    const bool ok = r_val <= 1e-12 * vb_norm || score <= accept_tol;
    rep.validated = ok;
    if (ok) return rep;
    if (score < best_score) {
      best_score = score;
      best = rep;
      have_best = true;
    }
  }
  if (!have_best) throw SketchRankFailure("solve_with_retries: all attempts rank deficient");
  best.validated = false;
  return best;
}

double residual_norm(const LsrProblem& p, const Vector& x) {  // lsr.cpp:26-28
  validate(p);
  DeviceMatrix dA = DeviceMatrix::upload(p.A);
  DevBuf<double> db(p.b), dx(x), out(2);
  check(slra_lsr_residual(device_context(), dA.data(), dA.ld(), p.A.rows(), p.A.cols(), db.get(), dx.get(),
                          out.get()),
        "residual_norm");
  return std::sqrt(out.download()[0]);
}

LsrReport sketch_solve(const LsrProblem& p, const SketchOperator& F, bool with_true_residual) {  // lsr.cpp:37-67
  validate(p);
  if (F.cols() != p.A.rows()) throw std::invalid_argument("sketch_solve: F cols != m");
  if (F.rows() <= p.A.cols()) throw std::invalid_argument("sketch_solve: need k > d");
  DeviceMatrix dA = DeviceMatrix::upload(p.A);
  DevBuf<double> db(p.b);
  LsrReport rep = sketch_solve_resident(dA, db.get(), F);
  if (with_true_residual) {
    rep.true_residual = residual_norm(p, rep.x_hat);
    rep.ratio = residual_ratio(p, rep.x_hat);
  }
  return rep;
}

Vector solve_exact(const LsrProblem& p) {  // lsr.cpp:21-24: pseudo_inverse(A) * b
  validate(p);
  DeviceMatrix dA = DeviceMatrix::upload(p.A);
  DevBuf<double> db(p.b), dx(static_cast<size_t>(p.A.cols()));
  int64_t rank = 0;
  check(slra_lsq_exact(device_context(), dA.data(), dA.ld(), p.A.rows(), p.A.cols(), db.get(), dx.get(), &rank),
        "solve_exact");
  return dx.download();
}

double residual_ratio(const LsrProblem& p, const Vector& x_hat) {  // lsr.cpp:30-35
  const double opt = residual_norm(p, solve_exact(p));
  double bn = 0;
  for (double x : p.b) bn += x * x;
  if (opt < 1e-14 * std::sqrt(bn)) return std::numeric_limits<double>::infinity();
  return residual_norm(p, x_hat) / opt;
}

LsrReport sketch_solve_sharded(slra_comm comm, const double* dA, Index lda, Index m_local, Index d, const double* db,
                               Index row0, Index m_global, const SketchOperator& F, bool with_true_residual) {
  if (!comm) throw std::invalid_argument("sketch_solve_sharded: no communicator");
  if (F.cols() != m_global) throw std::invalid_argument("sketch_solve: F cols != m");
  if (F.rows() <= d) throw std::invalid_argument("sketch_solve: need k > d");
  if (row0 < 0 || m_local < 0 || row0 + m_local > m_global || lda < m_local)
    throw std::invalid_argument("sketch_solve_sharded: bad row range");
  slra_ctx cx = device_context();
  const SketchPlan plan = compile_plan(F, Side::Left);
  if (plan.tree) throw std::invalid_argument("sketch_solve_sharded: butterfly (abridged Hadamard) plans do not shard");
  const Index k = plan.count;
  DevBuf<int64_t> src(plan.src);
  DevBuf<double> coef(plan.coef);
  // per-rank contributions to F (A | b): foreign rows are skipped (exact zeros)
  DevBuf<double> FW(static_cast<size_t>(k * (d + 1)));
  check(slra_sketch_rows_shard(cx, dA, lda, row0, m_local, d, src.get(), coef.get(), plan.width, k, FW.get(), k, 0),
        "sketch_solve_sharded");
  check(slra_sketch_rows_shard(cx, db, m_local, row0, m_local, 1, src.get(), coef.get(), plan.width, k,
                               FW.get() + k * d, k, 0),
        "sketch_solve_sharded");
  check(slra_comm_allreduce_sum(comm, FW.get(), FW.get(), k * (d + 1)), "sketch_solve_sharded: allreduce");
  DevBuf<double> dx(static_cast<size_t>(d));
  LsrReport rep;
  check(slra_lsr_solve_sketched(cx, FW.get(), k, k, d, dx.get(), &rep.sketched_residual), "sketch_solve");
  rep.x_hat = dx.download();
  rep.k = F.rows();
  if (with_true_residual) {
    DevBuf<double> out(2);
    check(slra_lsr_residual(cx, dA, lda, m_local, d, db, dx.get(), out.get()), "residual_norm");
    check(slra_comm_allreduce_sum(comm, out.get(), out.get(), 1), "residual_norm: allreduce");
    rep.true_residual = std::sqrt(out.download()[0]);
  }
  return rep;
}

}  // namespace slra
