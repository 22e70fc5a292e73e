// the SLRA_B200 definition of cross_approx (cur.hpp:70-73,
// cur.cpp:201-255) the reference's cur.cpp would carry — the C-ABI call and
// the copies back into the reference types. (stop_tol and the empty initial
// set's Rng draw are handled by the caller in this example.)
#include "ref_shim.hpp"

#include "b200.hpp"

namespace slra {

std::pair<CurDecomposition, CaTrace> cross_approx(const EntryOracle& M, Index r, Index k, Index l,
                                                  IndexSet init_rows, int loops, double h) {
  using namespace b200;
  const Index m = M.rows(), n = M.cols();
  if (init_rows.size() != k) throw std::invalid_argument("cross_approx: need k initial rows");
  const Matrix A = M.dense();
  Dev dA(8 * m * n), dI0(8 * k), dI(8 * k), dJ(8 * l), dU(8 * l * k), dTr(8 * 2 * loops * k),
      dTc(8 * 2 * loops * l), dTv(8 * 2 * loops);
  check(slra_memcpy_h2d(ctx(), dA.p, A.data(), 8 * m * n), "h2d");
  check(slra_memcpy_h2d(ctx(), dI0.p, init_rows.indices().data(), 8 * k), "h2d");
  int64_t r_used = 0;
  check(slra_cross_approx(ctx(), dA.as<double>(), m, m, n, r, k, l, dI0.as<int64_t>(), loops, h, dI.as<int64_t>(),
                          dJ.as<int64_t>(), dU.as<double>(), dTr.as<int64_t>(), dTc.as<int64_t>(), dTv.as<double>(),
                          nullptr, nullptr, &r_used),
        "cross_approx");
  std::vector<Index> I(k), J(l), tr(2 * loops * k), tc(2 * loops * l);
  std::vector<double> tv(2 * loops);
  CurDecomposition c;
  c.nucleus = Matrix(l, k);
  check(slra_memcpy_d2h(ctx(), I.data(), dI.p, 8 * k), "d2h");
  check(slra_memcpy_d2h(ctx(), J.data(), dJ.p, 8 * l), "d2h");
  check(slra_memcpy_d2h(ctx(), c.nucleus.data(), dU.p, 8 * l * k), "d2h");
  check(slra_memcpy_d2h(ctx(), tr.data(), dTr.p, 8 * 2 * loops * k), "d2h");
  check(slra_memcpy_d2h(ctx(), tc.data(), dTc.p, 8 * 2 * loops * l), "d2h");
  check(slra_memcpy_d2h(ctx(), tv.data(), dTv.p, 8 * 2 * loops), "d2h");
  c.row_set = IndexSet(I, m);
  c.col_set = IndexSet(J, n);
  c.r = r_used;
  CaTrace trace;
  for (int s = 0; s < 2 * loops; ++s) {
    CaStep st;
    st.horizontal = (s % 2) == 1;
    st.rows.assign(tr.begin() + s * k, tr.begin() + (s + 1) * k);
    st.cols.assign(tc.begin() + s * l, tc.begin() + (s + 1) * l);
    st.volume_proxy = tv[s];
    trace.steps.push_back(std::move(st));
  }
  return {std::move(c), std::move(trace)};
}

}  // namespace slra
