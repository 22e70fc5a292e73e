"""Config 4 (sketched least squares) at the BASELINE size and the LSR solve
semantics (lsr.cpp:21-67):

* full size: A 2^20 x 256 fp64 Gaussian, b = A x0 + 1e-6 e from the
  reference generator (gen_lsr_family pattern, testgen.cpp:159-193), 4096
  rows sampled uniformly and by the sparse +-1 sketch with 2 nonzeros per
  row; x_hat and the residual against the oracle's sketch_solve
  (ColPivHouseholderQR, threshold 1e-10) and the exact solution;
* the rank rule: sketches whose sigma_min / sigma_max sits between 1e-10
  and 1e-7 are SOLVED (the reference's ColPivQR rank is d), below 1e-10
  they raise SketchRankFailure, as the reference;
* d > 500 with the dominant column past index 500;
* solve_exact = pinv(A) b including rank-deficient A (minimum-norm
  solution), and residual_ratio.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slra():
    import paper_1611_01391_b200 as s
    return s


@pytest.fixture(scope="module")
def full_problem(slra, oracle):
    m, d = 1 << 20, 256
    A, b = slra.gen_lsr_gaussian(m, d, 1e-6, slra.Rng(2024))
    return A, b


def _samplers(mod, m, k, seed):
    ru = mod.Rng(mod.Rng.derive_seed(seed, 41))
    Fu = mod.make_sub_identity(ru.distinct_indices(k, m), m)
    rs = mod.Rng(mod.Rng.derive_seed(seed, 42))
    Fs = mod.make_product([mod.make_sub_identity(rs.distinct_indices(k, m), m), mod.gen_sparse_circulant(m, 2, rs),
                           mod.gen_sign_diagonal(m, rs)])
    return [("uniform_rows", Fu), ("sparse_pm1_s2", Fs)]


def test_config4_full_size_parity(slra, oracle, full_problem):
    A, b = full_problem
    m, d = A.shape
    Ao, bo = oracle.gen_lsr_gaussian(m, d, 1e-6, oracle.Rng(2024))
    assert np.array_equal(A, Ao) and np.array_equal(b, bo)
    nb = np.linalg.norm(b)
    xe = slra.solve_exact(A, b)
    # the oracle's solve_exact restates pinv through a one-sided Jacobi SVD of
    # the whole 2^20 x 256 A (minutes on the host); LAPACK's gelsd computes the
    # same minimum-norm solution with the same relative cut
    xeo = np.linalg.lstsq(A, b, rcond=1e-10)[0]
    assert np.linalg.norm(xe - xeo) <= 1e-10 * np.linalg.norm(xeo)
    opt = slra.residual_norm(A, b, xe)
    for (name, Fg), (_, Fo) in zip(_samplers(slra, m, 4096, 0), _samplers(oracle, m, 4096, 0)):
        g = slra.sketch_solve(A, b, Fg, False)
        o = oracle.sketch_solve(A, b, Fo, False)
        xo = o["x_hat"]
        assert np.linalg.norm(g["x_hat"] - xo) <= 1e-10 * np.linalg.norm(xo), name
        assert abs(g["sketched_residual"] - o["sketched_residual"]) <= 1e-8 * o["sketched_residual"], name
        rg = slra.residual_norm(A, b, g["x_hat"])
        ro = oracle.residual_norm(A, b, xo)
        assert abs(rg - ro) <= 1e-10 * nb, name
        ratio = rg / opt
        assert 1.0 <= ratio < 2.0, (name, ratio)
        print(f"config 4 {name}: residual ratio vs exact {ratio:.4f}")


def _conditioned(m, d, cond, seed):
    """A = U diag(s) V^T with s log-spaced from 1 to 1/cond; b = A x + noise."""
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, d)))
    V, _ = np.linalg.qr(rng.standard_normal((d, d)))
    s = np.logspace(0, -np.log10(cond), d)
    A = np.asfortranarray((U * s) @ V.T)
    b = A @ rng.standard_normal(d) + 1e-3 * rng.standard_normal(m)
    return A, b


@pytest.mark.parametrize("cond", [1e8, 1e9])
def test_near_deficient_sketch_solved_as_reference(slra, oracle, cond):
    """sigma_min / sigma_max in (1e-10, 1e-7): the reference's ColPivQR has
    full rank and solves; the device takes the exact path and agrees."""
    m, d, k = 6000, 40, 1200
    A, b = _conditioned(m, d, cond, 3)
    rows = slra.Rng(5).distinct_indices(k, m)
    g = slra.sketch_solve(A, b, slra.make_sub_identity(rows, m), False)
    o = oracle.sketch_solve(A, b, oracle.make_sub_identity(rows, m), False)
    # x_hat is determined to ~cond * eps relative; the sketched residual and
    # the true residual are well determined
    assert abs(g["sketched_residual"] - o["sketched_residual"]) <= 1e-6 * o["sketched_residual"]
    rg = slra.residual_norm(A, b, g["x_hat"])
    ro = oracle.residual_norm(A, b, o["x_hat"])
    assert abs(rg - ro) <= 1e-8 * ro
    assert np.linalg.norm(A @ (g["x_hat"] - o["x_hat"])) <= 1e-6 * np.linalg.norm(b)


@pytest.mark.parametrize("cond", [1e11, 1e13])
def test_deficient_sketch_raises_as_reference(slra, oracle, cond):
    m, d, k = 6000, 40, 1200
    A, b = _conditioned(m, d, cond, 4)
    rows = slra.Rng(6).distinct_indices(k, m)
    with pytest.raises(oracle.SketchRankFailure):
        oracle.sketch_solve(A, b, oracle.make_sub_identity(rows, m), False)
    with pytest.raises(slra.SketchRankFailure):
        slra.sketch_solve(A, b, slra.make_sub_identity(rows, m), False)


def test_wide_dominant_column_after_500(slra, oracle):
    """d = 600, the largest column at index 550 (1e7 x the others) and a
    near-dependent pair: the rank floor must come from all d columns."""
    rng = np.random.default_rng(8)
    m, d, k = 8000, 600, 2400
    A = rng.standard_normal((m, d))
    A[:, 550] *= 1e7
    A[:, 20] = A[:, 10] + 1e-9 * rng.standard_normal(m)
    A = np.asfortranarray(A)
    b = rng.standard_normal(m)
    rows = slra.Rng(9).distinct_indices(k, m)
    with pytest.raises(oracle.SketchRankFailure):
        oracle.sketch_solve(A, b, oracle.make_sub_identity(rows, m), False)
    with pytest.raises(slra.SketchRankFailure):
        slra.sketch_solve(A, b, slra.make_sub_identity(rows, m), False)


def test_solve_exact_rank_deficient_min_norm(slra, oracle):
    """solve_exact is pinv(A) b (lsr.cpp:21-24): a rank-deficient A gets the
    minimum-norm solution, never a rank failure; residual_ratio follows."""
    rng = np.random.default_rng(11)
    m, d = 3000, 24
    A = rng.standard_normal((m, d))
    A[:, 7] = A[:, 3]
    A[:, 19] = 2.0 * A[:, 5] - A[:, 11]
    A = np.asfortranarray(A)
    b = rng.standard_normal(m)
    xg = slra.solve_exact(A, b)
    xo = oracle.solve_exact(A, b)
    xn = np.linalg.pinv(A, rcond=1e-10) @ b
    assert np.linalg.norm(xo - xn) <= 1e-10 * np.linalg.norm(xn)
    assert np.linalg.norm(xg - xo) <= 1e-10 * np.linalg.norm(xo)
    x_try = xg + 0.01 * rng.standard_normal(d)
    assert abs(slra.residual_ratio(A, b, x_try) - oracle.residual_ratio(A, b, x_try)) <= 1e-10


def test_solve_exact_well_conditioned_fast_path(slra, oracle):
    rng = slra.Rng(21)
    A, b = slra.gen_lsr_gaussian(50000, 64, 1e-3, rng)
    xg = slra.solve_exact(A, b)
    xo = oracle.solve_exact(A, b)
    assert np.linalg.norm(xg - xo) <= 1e-10 * np.linalg.norm(xo)


@pytest.mark.parametrize("d,k", [(1, 64), (7, 300), (32, 512), (33, 700), (100, 1500), (255, 4096), (256, 4096),
                                 (256, 65536)])
def test_cluster_solve_shapes_vs_oracle(slra, oracle, d, k):
    """The d <= 256 fast path (augmented Gram on DMMA, Cholesky + solve +
    refinement on one 8-CTA cluster) on ragged panel counts (d not a
    multiple of 32, one panel, a single column) and k up to the cluster
    path's limit: x_hat and the sketched residual within 1e-10 of the
    oracle's ColPivHouseholderQR solve (lsr.cpp:52-60)."""
    rng = np.random.default_rng(d * 1000 + k)
    m = max(2 * k, 4 * d)
    A = np.asfortranarray(rng.standard_normal((m, d)) * np.exp(rng.uniform(-2, 2, d)))
    b = A @ rng.standard_normal(d) + 1e-3 * rng.standard_normal(m)
    rows = slra.Rng(d + k).distinct_indices(k, m)
    g = slra.sketch_solve(A, b, slra.make_sub_identity(rows, m), False)
    o = oracle.sketch_solve(A, b, oracle.make_sub_identity(rows, m), False)
    xo = o["x_hat"]
    assert np.linalg.norm(g["x_hat"] - xo) <= 1e-10 * np.linalg.norm(xo)
    assert abs(g["sketched_residual"] - o["sketched_residual"]) <= 1e-10 * max(o["sketched_residual"], 1e-300) + \
        1e-12 * np.linalg.norm(b)


def test_residual_multi_matches_single(slra):
    """slra_lsr_residual_multi: ||A x_s - b||^2 for two and four solutions in
    one pass equals the one-solution pass bit for bit (same per-thread order)."""
    import torch
    rng = np.random.default_rng(11)
    m, d = 100003, 67  # odd m: the scalar tail rows
    A = torch.from_numpy(np.asfortranarray(rng.standard_normal((m, d))).T.copy()).cuda()  # A^T rows = columns of A
    b = torch.from_numpy(rng.standard_normal(m)).cuda()
    for nx in (2, 4):
        X = torch.from_numpy(rng.standard_normal((nx, d))).cuda()
        out = torch.zeros(nx, dtype=torch.float64, device="cuda")
        slra.lsr_residual_multi_device(A.data_ptr(), m, m, d, b.data_ptr(), X.data_ptr(), nx, out.data_ptr())
        for s in range(nx):
            one = torch.zeros(1, dtype=torch.float64, device="cuda")
            slra.lsr_residual_device(A.data_ptr(), m, m, d, b.data_ptr(), X[s].data_ptr(), one.data_ptr())
            assert out[s].item() == one.item()
            ref = torch.linalg.vector_norm(A.T @ X[s] - b).item() ** 2
            assert abs(out[s].item() - ref) <= 1e-12 * ref


def test_sketch_solve_batched_matches_separate_calls(slra):
    """slra_sketch_solve_batched (a cluster per sketch, one launch) gives the
    bits of separate slra_sketch_solve calls, for the config-4 sampler kinds
    and for a sketch that takes the exact (ColPivQR) path."""
    import torch
    rng = np.random.default_rng(31)
    m, d, k = 40000, 96, 1024
    A = np.asfortranarray(rng.standard_normal((m, d)))
    A[:, 7] = A[:, 3] + 1e-9 * rng.standard_normal(m)  # near-dependent pair: the exact path for every sketch
    for near in (False, True):
        Ause = A if near else np.asfortranarray(rng.standard_normal((m, d)))
        b = Ause @ rng.standard_normal(d) + 1e-3 * rng.standard_normal(m)
        At = torch.from_numpy(Ause.T.copy()).cuda()
        bd = torch.from_numpy(b).cuda()
        plans = []
        for F in (slra.make_sub_identity(slra.Rng(5).distinct_indices(k, m), m),
                  slra.make_product([slra.make_sub_identity(slra.Rng(6).distinct_indices(k, m), m),
                                     slra.gen_sparse_circulant(m, 2, slra.Rng(7)), slra.gen_sign_diagonal(m, slra.Rng(8))])):
            p = F.plan("left")
            plans.append((p, torch.tensor(p["src"], dtype=torch.int64, device="cuda"),
                          torch.tensor(p["coef"], dtype=torch.float64, device="cuda"),
                          torch.tensor(p["q"], dtype=torch.int32, device="cuda")))
        xs = [torch.zeros(d, dtype=torch.float64, device="cuda") for _ in plans]
        xb = [torch.zeros(d, dtype=torch.float64, device="cuda") for _ in plans]
        sep = [slra.sketch_solve_device(At.data_ptr(), m, m, d, bd.data_ptr(), s.data_ptr(), c.data_ptr(), q.data_ptr(),
                                        p["width"], p["tree"], k, x.data_ptr()) for (p, s, c, q), x in zip(plans, xs)]
        bat = slra.sketch_solve_batched_device(At.data_ptr(), m, m, d, bd.data_ptr(), [s.data_ptr() for _, s, _, _ in plans],
                                               [c.data_ptr() for _, _, c, _ in plans], [q.data_ptr() for *_, q in plans],
                                               [p["width"] for p, *_ in plans], [p["tree"] for p, *_ in plans], k,
                                               [x.data_ptr() for x in xb])
        torch.cuda.synchronize()
        assert list(sep) == list(bat)
        for a_, b_ in zip(xs, xb):
            assert torch.equal(a_, b_)
