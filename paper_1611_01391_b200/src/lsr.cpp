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
}  // namespace

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
  const Index d = p.A.cols(), m = p.A.rows();
  if (F.cols() != m) throw std::invalid_argument("sketch_solve: F cols != m");
  if (F.rows() <= d) throw std::invalid_argument("sketch_solve: need k > d");
  const SketchPlan plan = compile_plan(F, Side::Left);
  DeviceMatrix dA = DeviceMatrix::upload(p.A);
  DevBuf<double> db(p.b), dx(static_cast<size_t>(d));
  DevBuf<int64_t> src(plan.src);
  DevBuf<double> coef(plan.coef);
  DevBuf<int32_t> q(plan.q);
  LsrReport rep;
  check(slra_sketch_solve(device_context(), dA.data(), dA.ld(), m, d, db.get(), src.get(), coef.get(), q.get(),
                          plan.width, plan.tree, plan.count, dx.get(), &rep.sketched_residual),
        "sketch_solve");
  rep.x_hat = dx.download();
  rep.k = F.rows();
  if (with_true_residual) {
    rep.true_residual = residual_norm(p, rep.x_hat);
    rep.ratio = residual_ratio(p, rep.x_hat);
  }
  return rep;
}

Vector solve_exact(const LsrProblem& p) {  // lsr.cpp:21-24 (device normal-equation solve)
  validate(p);
  // exact LS = sketch_solve with the identity sketch (all m rows, in order)
  std::vector<Index> all(static_cast<size_t>(p.A.rows()));
  for (Index i = 0; i < p.A.rows(); ++i) all[static_cast<size_t>(i)] = i;
  const auto F = make_sub_identity(IndexSet(all, p.A.rows()), p.A.rows());
  return sketch_solve(p, *F, false).x_hat;
}

double residual_ratio(const LsrProblem& p, const Vector& x_hat) {  // lsr.cpp:30-35
  const double opt = residual_norm(p, solve_exact(p));
  double bn = 0;
  for (double x : p.b) bn += x * x;
  if (opt < 1e-14 * std::sqrt(bn)) return std::numeric_limits<double>::infinity();
  return residual_norm(p, x_hat) / opt;
}

}  // namespace slra
