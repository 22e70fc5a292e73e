"""Range-finder variants: pseudo_inverse, lra_premult and
two_stage_truncate on the B200 against the oracle (needs a GPU: `-m gpu`).

Properties restate /root/reference/proj/tests/test_lra.cpp:98-193 on the
product; parity cases compare with the oracle on the same seeded inputs, with
the sketches drawn from each library's own Rng (same stream). Factors are
compared through their products, which are unique (the bases differ by
rounding only); tolerance 1e-10 relative (north_star).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def slra():
    import paper_1611_01391_b200 as s
    return s


def spec(A):
    return np.linalg.norm(A, 2)


# ---------------------------------------------------------------- pseudo-inverse
@pytest.mark.parametrize("shape", [(5, 3), (3, 5), (64, 64), (300, 48), (48, 300), (4096, 20)])
def test_pinv_vs_oracle(slra, oracle, shape):  # linalg.cpp:111-121
    A = oracle.Rng(40 + sum(shape)).gaussian_matrix(*shape)
    P = slra.pseudo_inverse(A, 1e-10)
    Po = oracle.pseudo_inverse(A, 1e-10)
    assert P.shape == (shape[1], shape[0])
    assert np.linalg.norm(P - Po) <= TOL * np.linalg.norm(Po) * 10


def test_pinv_known_answers(slra):  # test_linalg.cpp:150-169
    rng = slra.Rng(9)
    Q, _ = slra.thin_qr(rng.gaussian_matrix(4, 4))
    assert np.linalg.norm(slra.pseudo_inverse(Q, 1e-10) - Q.T) < 1e-12
    Dp = slra.pseudo_inverse(np.diag([2.0, 0.0]), 1e-8)
    assert Dp[0, 0] == pytest.approx(0.5) and Dp[1, 1] == 0.0 and Dp[0, 1] == 0.0
    assert np.linalg.norm(slra.pseudo_inverse(np.zeros((3, 2)), 1e-10)) == 0.0
    # rank-deficient: the cut drops the null direction
    A = rng.gaussian_matrix(7, 2) @ rng.gaussian_matrix(2, 5)
    assert np.allclose(slra.pseudo_inverse(A, 1e-10), np.linalg.pinv(A, rcond=1e-10), atol=1e-12)


# ---------------------------------------------------------------- lra_premult
def test_premult_identity_matches_range_finder(slra):  # test_lra.cpp:98-108
    rng = slra.Rng(25)
    m, n = 30, 24
    M = rng.gaussian_matrix(m, n)
    H = slra.gen_gaussian(n, 6, rng)
    F = slra.make_sub_identity(list(range(m)), m)
    Ua, Va = slra.range_finder(M, H, 4)
    Ub, Vb = slra.lra_premult(M, F, H, 4)
    assert spec(Ua - Ub) <= 1e-12
    assert spec(Va - Vb) <= 1e-12


def test_premult_exact_rank(slra):  # test_lra.cpp:110-120
    for t in range(10):
        rng = slra.Rng(900 + t)
        m, n, r, l, k = 48, 40, 5, 8, 12
        M = slra.gen_factor_gaussian(m, n, r, 0.0, rng)
        H = slra.gen_gaussian(n, l, rng)
        F = slra.gen_gaussian(k, m, rng)
        U, V = slra.lra_premult(M, F, H, r)
        assert spec(M - U @ V) <= 1e-9 * spec(M)


def test_premult_residual_identity_and_impact(slra):  # test_lra.cpp:122-142
    rng = slra.Rng(26)
    m, n, r, l, k = 8, 8, 2, 3, 5
    for _ in range(20):
        M = rng.gaussian_matrix(m, n)
        Hd = rng.gaussian_matrix(n, l)
        Fd = rng.gaussian_matrix(k, m)
        U, V = slra.lra_premult(M, slra.make_gaussian(Fd), slra.make_gaussian(Hd), r)
        FU = Fd @ U
        FUp = np.linalg.pinv(FU, rcond=1e-10)
        P = np.eye(m) - U @ FUp @ Fd
        resid = P @ (M - U @ (U.T @ M))
        assert spec(M - U @ V - resid) <= 1e-9 * spec(M)
        assert spec(P) <= (1 + spec(U) * spec(FUp) * spec(Fd)) * (1 + 1e-12)


def test_premult_rank_failure(slra):  # test_lra.cpp:144-150
    rng = slra.Rng(27)
    M = slra.gen_factor_gaussian(16, 16, 3, 0.0, rng)
    H = slra.gen_gaussian(16, 4, rng)
    F = slra.make_gaussian(np.zeros((5, 16)))
    with pytest.raises(slra.PremultRankFailure):
        slra.lra_premult(M, F, H, 3)
    # the range check still comes first (lra.cpp:45 -> RangeFailure)
    with pytest.raises(slra.RangeFailure):
        slra.lra_premult(np.zeros((16, 16)), slra.gen_gaussian(5, 16, rng), H, 1)


def test_premult_invalid_arguments(slra):
    rng = slra.Rng(3)
    M = rng.gaussian_matrix(20, 12)
    H = slra.gen_gaussian(12, 4, rng)
    with pytest.raises(ValueError):
        slra.lra_premult(M, slra.gen_gaussian(5, 19, rng), H, 2)  # F cols != m
    with pytest.raises(ValueError):
        slra.lra_premult(M, slra.gen_gaussian(5, 20, rng), H, 5)  # r > l


@pytest.mark.parametrize("truncated", [False, True])
@pytest.mark.parametrize("m,n,l,s,r", [(300, 200, 12, 40, 5), (4096, 1024, 48, 256, 20)])
def test_premult_structured_vs_oracle(slra, oracle, truncated, m, n, l, s, r):
    """Config-2-style sketches on both sides: H = sparse circulant column
    slice (right plan), F = SubIdentity(s of m) Z_f D (left plan)."""
    seed = 4000 + m + l + truncated
    M = oracle.gen_factor_gaussian(m, n, r, 1e-6, oracle.Rng(seed))
    rp, ro = slra.Rng(seed + 1), oracle.Rng(seed + 1)
    Hp = slra.take_columns_random(slra.gen_sparse_circulant(n, 4, rp), l, rp)
    Ho = oracle.take_columns_random(oracle.gen_sparse_circulant(n, 4, ro), l, ro)
    sp, so = rp.distinct_indices(s, m), ro.distinct_indices(s, m)
    Fp = slra.make_product([slra.make_sub_identity(sp, m), slra.gen_sparse_circulant(m, 2, rp),
                            slra.gen_sign_diagonal(m, rp)])
    Fo = oracle.make_product([oracle.make_sub_identity(so, m), oracle.gen_sparse_circulant(m, 2, ro),
                              oracle.gen_sign_diagonal(m, ro)])
    U, V = slra.lra_premult(M, Fp, Hp, r, truncated)
    Uo, Vo = oracle.lra_premult(M, Fo, Ho, r, truncated)
    assert U.shape == Uo.shape and V.shape == Vo.shape
    nM = np.linalg.norm(M)
    assert np.linalg.norm(U @ V - Uo @ Vo) <= TOL * nM
    # same residual as the oracle, and near the range finder's own
    e, eo = np.linalg.norm(M - U @ V), np.linalg.norm(M - Uo @ Vo)
    assert abs(e - eo) <= TOL * nM
    if truncated:  # U = S_r Sigma_r is unique up to column signs (sign rule fixes them)
        assert np.linalg.norm(U - Uo) <= TOL * nM


# ---------------------------------------------------------------- two_stage_truncate
def test_two_stage_truncate_known_answers(slra):  # test_lra.cpp:152-170
    rng = slra.Rng(28)
    m, n, l = 40, 32, 8
    U = rng.gaussian_matrix(m, l)
    V = rng.gaussian_matrix(l, n)
    P = U @ V
    Us, Vs = slra.two_stage_truncate(U, V, l)
    assert spec(P - Us @ Vs) <= 1e-12 * spec(P)
    U3, V3 = slra.two_stage_truncate(U, V, 3)
    S, sig, Tt = np.linalg.svd(P)
    assert spec(U3 @ V3 - (S[:, :3] * sig[:3]) @ Tt[:3]) <= 1e-9 * spec(P)
    with pytest.raises(ValueError):
        slra.two_stage_truncate(U, V, l + 1)


def test_two_stage_truncation_bound(slra):  # test_lra.cpp:172-193 (all 100 trials)
    for t in range(100):
        rng = slra.Rng(1000 + t)
        n, r, l = 64, 4, 8
        M = slra.gen_factor_gaussian(n, n, r, 1e-4, rng)
        H = slra.gen_gaussian(n, l, rng)
        U, V = slra.range_finder(M, H, r)
        Ug, Vg = slra.two_stage_truncate(U, V, r)
        sig = np.linalg.svd(M, compute_uv=False)
        tau = np.sqrt(np.sum(sig[r:] ** 2))
        assert np.linalg.norm(M - Ug @ Vg) <= (tau + 2 * np.linalg.norm(M - U @ V)) * (1 + 1e-8)


@pytest.mark.parametrize("m,n,l,r", [(40, 32, 8, 3), (4096, 2048, 48, 20), (1000, 30, 30, 30), (70, 700, 64, 10)])
def test_two_stage_truncate_vs_oracle(slra, oracle, m, n, l, r):
    rng = oracle.Rng(77 + m + r)
    U = rng.gaussian_matrix(m, l)
    V = rng.gaussian_matrix(l, n)
    Ug, Vg = slra.two_stage_truncate(U, V, r)
    Uo, Vo = oracle.two_stage_truncate(U, V, r)
    assert Ug.shape == (m, r) and Vg.shape == (r, n)
    nP = np.linalg.norm(U @ V)
    # both factors are unique given the svd sign rule (distinct singular values)
    assert np.linalg.norm(Ug - Uo) <= TOL * nP
    assert np.linalg.norm(Vg - Vo) <= 1e-9 * np.sqrt(r)
    assert np.linalg.norm(Ug @ Vg - Uo @ Vo) <= TOL * nP
