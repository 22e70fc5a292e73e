"""Pin the CPU oracle (oracle/, test infrastructure) before trusting it.

Every known-answer test the reference holds for the hot path
is restated here against the oracle, plus the C++ standard's mt19937_64 value
and LAPACK (scipy) cross-checks. Reference citations are
/root/reference/proj/tests/<file>:<line>.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla


# ---------------------------------------------------------------- Rng
def test_mt19937_64_standard_value(oracle):
    # [rand.predef]: the 10000th draw of a default-seeded mt19937_64.
    r = oracle.Rng(5489)
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042


def test_rng_determinism(oracle):  # test_linalg.cpp:243-251
    a, b = oracle.Rng(42), oracle.Rng(42)
    assert [a.gaussian() for _ in range(100)] == [b.gaussian() for _ in range(100)]
    assert np.array_equal(oracle.Rng(7).gaussian_matrix(4, 4), oracle.Rng(7).gaussian_matrix(4, 4))
    assert oracle.Rng(9).permutation(10) == oracle.Rng(9).permutation(10)


def test_rng_formulas(oracle):
    # rng.hpp:21-23: uniform = (u64 >> 11) * 2^-53; rng.cpp:60-66 splitmix.
    r1, r2 = oracle.Rng(3), oracle.Rng(3)
    u = r1.uniform()
    assert u == (r2.next_u64() >> 11) * 2.0**-53
    z = (0 + 0x9E3779B97F4A7C15 * 1) % 2**64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % 2**64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % 2**64
    assert oracle.Rng.derive_seed(0, 0) == z ^ (z >> 31)
    # gaussian: Box-Muller cos branch (rng.cpp:8-14)
    r1, r2 = oracle.Rng(11), oracle.Rng(11)
    g = r1.gaussian()
    u1 = r2.uniform()
    u2 = r2.uniform()
    assert g == math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)
    # distinct_indices: partial Fisher-Yates, distinct and in range
    d = oracle.Rng(5).distinct_indices(64, 100)
    assert len(set(d)) == 64 and min(d) >= 0 and max(d) < 100
    p = oracle.Rng(5).permutation(50)
    assert sorted(p) == list(range(50))


# ---------------------------------------------------------------- QR / SVD
def test_thin_qr_known_answer(oracle):  # test_linalg.cpp:45-52
    Q, R = oracle.thin_qr(np.array([[3.0], [4.0]]))
    assert Q[0, 0] == pytest.approx(0.6) and Q[1, 0] == pytest.approx(0.8)
    assert R[0, 0] == pytest.approx(5.0)


def test_thin_qr_invariants(oracle):  # test_linalg.cpp:53-68
    B = oracle.Rng(7).gaussian_matrix(8, 3)
    Q, R = oracle.thin_qr(B)
    assert np.linalg.norm(Q.T @ Q - np.eye(3)) <= 1e-13
    assert np.linalg.norm(Q @ R - B) <= 1e-12 * np.linalg.norm(B)
    assert (np.diag(R) >= 0).all()
    with pytest.raises(ValueError):
        oracle.thin_qr(np.zeros((2, 3)))
    # agrees with LAPACK up to the sign convention
    Qs, Rs = np.linalg.qr(B)
    s = np.sign(np.diag(Rs))
    assert np.allclose(Q, Qs * s, atol=1e-13)


def test_svd_examples(oracle):  # test_linalg.cpp:70-98
    S, sig, T = oracle.svd(np.diag([3.0, 1.0]))
    assert sig[0] == pytest.approx(3) and sig[1] == pytest.approx(1)
    assert np.linalg.norm(np.abs(S) - np.eye(2)) < 1e-12
    rng = oracle.Rng(3)
    u, v = rng.gaussian_vector(6), rng.gaussian_vector(4)
    S, sig, T = oracle.svd(np.outer(u, v))
    assert sig[0] == pytest.approx(np.linalg.norm(u) * np.linalg.norm(v))
    assert (sig[1:] <= 1e-13 * sig[0]).all()
    A = rng.gaussian_matrix(6, 4)
    S, sig, T = oracle.svd(A)
    lam = np.linalg.eigvalsh(A.T @ A)[::-1]
    assert np.allclose(sig, np.sqrt(lam), rtol=1e-10)
    assert np.linalg.norm(S @ np.diag(sig) @ T.T - A) <= 1e-12 * np.linalg.norm(A) * 4
    assert np.linalg.norm(S.T @ S - np.eye(4)) <= 4e-12
    assert np.linalg.norm(T.T @ T - np.eye(4)) <= 4e-12


def test_svd_sign_convention(oracle):  # test_linalg.cpp:100-109
    S, sig, T = oracle.svd(oracle.Rng(19).gaussian_matrix(7, 5))
    for j in range(S.shape[1]):
        assert S[np.argmax(np.abs(S[:, j])), j] >= 0


@pytest.mark.parametrize("shape", [(50, 7), (7, 50), (64, 64), (300, 48)])
def test_svd_vs_lapack(oracle, shape):
    A = oracle.Rng(sum(shape)).gaussian_matrix(*shape)
    S, sig, T = oracle.svd(A)
    assert np.allclose(sig, np.linalg.svd(A, compute_uv=False), rtol=1e-12, atol=1e-13 * sig[0])
    assert np.linalg.norm(S @ np.diag(sig) @ T.T - A) <= 1e-12 * np.linalg.norm(A) * 8


def test_pseudo_inverse(oracle):  # test_linalg.cpp:150-169
    rng = oracle.Rng(9)
    Q, _ = oracle.thin_qr(rng.gaussian_matrix(4, 4))
    assert np.linalg.norm(oracle.pseudo_inverse(Q) - Q.T) < 1e-12
    Dp = oracle.pseudo_inverse(np.diag([2.0, 0.0]), 1e-8)
    assert Dp[0, 0] == pytest.approx(0.5) and Dp[1, 1] == 0.0
    A = rng.gaussian_matrix(5, 3)
    Ap = oracle.pseudo_inverse(A)
    assert np.linalg.norm(A @ Ap @ A - A) <= 1e-11 * np.linalg.norm(A)
    assert np.linalg.norm(Ap @ A @ Ap - Ap) <= 1e-11 * np.linalg.norm(Ap)
    assert np.linalg.norm(A @ Ap - (A @ Ap).T) <= 1e-11
    assert np.linalg.norm(oracle.pseudo_inverse(np.zeros((3, 2)))) == 0.0


def test_numerical_rank(oracle):  # test_linalg.cpp:171-179
    D = np.diag([1.0, 1e-10])
    assert oracle.numerical_rank(D, 1e-6) == 1
    assert oracle.numerical_rank(np.zeros((3, 3)), 1e-6) == 0
    assert oracle.numerical_rank(D, 1e-6, True) == 1
    assert oracle.numerical_rank(D, 1e-11, True) == 2
    with pytest.raises(ValueError):
        oracle.numerical_rank(D, 0.0)


@pytest.mark.parametrize("shape", [(6, 40), (16, 256), (32, 256), (48, 300)])
def test_colpiv_pivots_match_lapack_geqp3(oracle, shape):
    # Eigen ColPivHouseholderQR follows LAPACK xGEQP3's pivot rule and norm
    # downdate; on generic inputs the pivot order must agree with dgeqp3.
    A = oracle.Rng(100 + shape[1]).gaussian_matrix(*shape)
    d = oracle.colpiv_qr(A)
    _, _, piv = sla.qr(A, pivoting=True, mode="economic")
    k = min(shape)
    assert list(d["perm"][:k]) == list(piv[:k])
    assert d["rank"] == k


def test_colpiv_solve(oracle):
    rng = oracle.Rng(77)
    A = rng.gaussian_matrix(20, 6)
    B = rng.gaussian_matrix(20, 3)
    X = oracle.colpiv_solve(A, B, 1e-10)
    Xs = np.linalg.lstsq(A, B, rcond=None)[0]
    assert np.allclose(X, Xs, atol=1e-12)
    G = rng.gaussian_matrix(5, 5)
    assert np.allclose(oracle.colpiv_solve(G, np.eye(5)), np.linalg.inv(G), atol=1e-11)


def test_index_set_validation(oracle):  # test_linalg.cpp:226-241 (through primitive_cur)
    M = np.arange(9.0).reshape(3, 3)
    with pytest.raises(ValueError):
        oracle.primitive_cur(M, [0, 0], [1, 2], 1)
    with pytest.raises(ValueError):
        oracle.primitive_cur(M, [3], [1], 1)


# ---------------------------------------------------------------- maxvol / CUR
def test_t_factor(oracle):  # test_cur.cpp:11-14
    assert oracle.t_factor(5, 5, 1.1) == pytest.approx(1.0)
    assert oracle.t_factor(10, 2, 1.0) == pytest.approx(math.sqrt(17.0))


def test_maxvol_known_answers(oracle):  # test_cur.cpp:16-33
    A = np.zeros((9, 3))
    A[0, 0] = A[1, 1] = A[2, 2] = 1.0
    assert set(oracle.maxvol_rows(A)) >= {0, 1, 2}
    assert oracle.maxvol_rows(np.array([[1.0], [2.0], [-3.0]]), 1.0) == [2]
    with pytest.raises(oracle.SelectionFailure):
        oracle.maxvol_rows(np.zeros((5, 2)))


def test_maxvol_dominance_and_volume(oracle):  # test_cur.cpp:35-60
    rng = oracle.Rng(31)
    m, r, h = 64, 4, 1.1
    A, _ = oracle.thin_qr(rng.gaussian_matrix(m, r))
    I = oracle.maxvol_rows(A, h)
    G = A[I, :]
    B = A @ np.linalg.inv(G)
    assert np.abs(B).max() <= h * (1 + 1e-12)
    assert np.linalg.norm(np.linalg.inv(G), 2) <= oracle.t_factor(m, r, h) * (1 + 1e-6)
    vol = abs(np.linalg.det(G))
    beaten = sum(vol >= abs(np.linalg.det(A[rng.distinct_indices(r, m), :])) for _ in range(1000))
    assert beaten >= 990


def test_primitive_cur_exact_rank(oracle):  # test_cur.cpp:62-78
    ok = failures = 0
    for t in range(100):
        rng = oracle.Rng(1300 + t)
        n, r = 48, 4
        M = oracle.gen_factor_gaussian(n, n, r, 0.0, rng)
        try:
            c = oracle.primitive_cur(M, rng.distinct_indices(r, n), rng.distinct_indices(r, n), r)
            err = np.linalg.norm(M - oracle.cur_reconstruct(M, c["I"], c["J"], c["nucleus"]), 2)
            ok += err <= 1e-8 * np.linalg.norm(M, 2)
        except oracle.GeneratorRankFailure:
            failures += 1
    assert ok >= 95 and ok + failures == 100


def test_primitive_cur_leading_block(oracle):  # test_cur.cpp:80-87
    M = np.diag([5.0, 4, 3, 2, 1, 0.5])
    c = oracle.primitive_cur(M, [0, 1, 2], [0, 1, 2], 3)
    R = oracle.cur_reconstruct(M, c["I"], c["J"], c["nucleus"])
    assert np.linalg.norm(R[:3, :3] - M[:3, :3]) <= 1e-12


def test_primitive_cur_missed_delta(oracle):  # test_cur.cpp:89-100
    D = np.zeros((8, 8))
    D[5, 5] = 1.0
    with pytest.raises(oracle.GeneratorRankFailure):
        oracle.primitive_cur(D, [0, 1], [0, 1], 1)
    Dp = D + 1e-8
    c = oracle.primitive_cur(Dp, [0, 1], [0, 1], 1)
    assert oracle.cur_evaluate(Dp, c["I"], c["J"], c["nucleus"], "chebyshev") >= 0.5


def test_primitive_cur_reads_only_generator(oracle):  # test_cur.cpp:101-108
    rng = oracle.Rng(32)
    M = oracle.gen_factor_gaussian(40, 30, 3, 0.0, rng)
    c = oracle.primitive_cur(M, rng.distinct_indices(5, 40), rng.distinct_indices(4, 30), 3)
    assert c["accesses"] == 20


def test_cross_approx_exactness_and_accounting(oracle):  # test_cur.cpp:145-155
    rng = oracle.Rng(35)
    m, n, r = 64, 48, 5
    M = oracle.gen_factor_gaussian(m, n, r, 0.0, rng)
    c = oracle.cross_approx(M, r, r, r, [], 1, 1.1, None, rng)
    err = np.linalg.norm(M - oracle.cur_reconstruct(M, c["I"], c["J"], c["nucleus"]), 2)
    assert err <= 1e-9 * np.linalg.norm(M, 2)
    assert len(c["trace"]) == 2
    assert c["accesses"] <= r * n + m * r + 2 * r * r


def test_cross_approx_extra_loops(oracle):  # test_cur.cpp:169-183 (reduced to 30 trials)
    ok = 0
    for t in range(30):
        M = oracle.gen_factor_gaussian(96, 96, 6, 1e-6, oracle.Rng(1600 + t))
        c1 = oracle.cross_approx(M, 6, 6, 6, [], 1, 1.1, None, oracle.Rng(1700 + t))
        c5 = oracle.cross_approx(M, 6, 6, 6, [], 5, 1.1, None, oracle.Rng(1700 + t))
        e1 = oracle.cur_evaluate(M, c1["I"], c1["J"], c1["nucleus"])
        e5 = oracle.cur_evaluate(M, c5["I"], c5["J"], c5["nucleus"])
        ok += e5 <= e1 * (1 + 1e-6)
    assert ok >= 27


def test_cross_approx_early_stop(oracle):  # test_cur.cpp:185-192
    rng = oracle.Rng(36)
    M = oracle.gen_factor_gaussian(64, 64, 4, 0.0, rng)
    c = oracle.cross_approx(M, 4, 4, 4, [], 8, 1.1, 1e-8, rng)
    assert len(c["trace"]) < 16
    assert c["trace"][-1]["error_estimate"] is not None


def test_cur_evaluate_norm_ordering(oracle):  # test_cur.cpp:194-205
    rng = oracle.Rng(37)
    M = oracle.gen_factor_gaussian(24, 24, 3, 1e-3, rng)
    c = oracle.primitive_cur(M, rng.distinct_indices(3, 24), rng.distinct_indices(3, 24), 3)
    sp = oracle.cur_evaluate(M, c["I"], c["J"], c["nucleus"], "spectral")
    fr = oracle.cur_evaluate(M, c["I"], c["J"], c["nucleus"], "frobenius")
    ch = oracle.cur_evaluate(M, c["I"], c["J"], c["nucleus"], "chebyshev")
    assert ch <= fr * (1 + 1e-12) and sp <= fr * (1 + 1e-12) and fr > 0


# ---------------------------------------------------------------- sketch operators
H4 = np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]], float)


def test_abridged_hadamard_displays(oracle):  # test_sketch.cpp:29-48
    E1 = np.array([[1, 0, 1, 0], [0, 1, 0, 1], [1, 0, -1, 0], [0, 1, 0, -1]], float)
    assert np.array_equal(oracle.materialize(oracle.make_abridged_hadamard(4, 1)), E1)
    assert np.array_equal(oracle.materialize(oracle.make_abridged_hadamard(4, 2)), H4)
    H8 = np.block([[H4, H4], [H4, -H4]])
    assert np.array_equal(oracle.materialize(oracle.make_abridged_hadamard(8, 3)), H8)
    with pytest.raises(ValueError):
        oracle.make_abridged_hadamard(6, 2)


def test_permutation_and_sign(oracle):  # test_sketch.cpp:79-96
    P = oracle.materialize(oracle.make_permutation([3, 2, 1, 0]))
    assert all(P[i, 3 - i] == 1.0 for i in range(4)) and P.sum() == 4.0
    rng = oracle.Rng(1)
    op = oracle.gen_permutation(8, rng)
    X = rng.gaussian_matrix(8, 3)
    assert np.array_equal(op.apply_transpose(op.apply(X)), X)
    D = oracle.materialize(oracle.gen_sign_diagonal(8, rng))
    assert np.array_equal(D @ D, np.eye(8))
    with pytest.raises(ValueError):
        oracle.make_sign_diagonal(np.zeros(3))


def test_sparse_circulant_dense_oracle(oracle):  # test_sketch.cpp:101-117
    rng = oracle.Rng(2)
    n, s = 16, 3
    op = oracle.gen_sparse_circulant(n, s, rng)
    Z = oracle.materialize(op)
    v = Z[:, 0]
    f = 0.0
    for i in range(1, n):
        if Z[0, i] != 0:
            f = Z[0, i] / v[n - i]
    Zo = np.array([[v[i - j] if i >= j else f * v[n + i - j] for j in range(n)] for i in range(n)])
    assert np.array_equal(Z, Zo)
    assert all((Z[:, j] != 0).sum() == s for j in range(n))
    X = rng.gaussian_matrix(n, 5)
    assert np.linalg.norm(op.apply(X) - Z @ X) < 1e-13 * np.linalg.norm(Z) * np.linalg.norm(X)
    assert np.linalg.norm(op.apply_transpose(X) - Z.T @ X) < 1e-13 * np.linalg.norm(Z) * np.linalg.norm(X)


def test_sub_identity_and_product(oracle):  # test_sketch.cpp:159-182
    op = oracle.make_sub_identity([1, 3], 4)
    M = np.array([[1, 2], [3, 4], [5, 6], [7, 8]], float)
    S = op.apply(M)
    assert S[0, 0] == 3.0 and S[1, 1] == 8.0
    assert (op.apply_transpose(S)[0] == 0).all()
    rng = oracle.Rng(7)
    prod = oracle.make_product([oracle.gen_permutation(8, rng), oracle.gen_sign_diagonal(8, rng),
                                oracle.make_abridged_hadamard(8, 2)])
    Pm = oracle.materialize(prod)
    X = rng.gaussian_matrix(8, 3)
    sc = 1e-13 * np.linalg.norm(Pm) * np.linalg.norm(X)
    assert np.linalg.norm(prod.apply(X) - Pm @ X) < sc
    assert np.linalg.norm(prod.apply_transpose(X) - Pm.T @ X) < sc


def test_asph_orthogonal_up_to_2d(oracle):  # test_sketch.cpp:185-190
    A = oracle.materialize(oracle.gen_asph(16, 2, oracle.Rng(8)))
    assert np.linalg.norm(A.T @ A - 4.0 * np.eye(16)) < 1e-11


def test_take_columns(oracle):  # test_sketch.cpp:192-203
    S = oracle.materialize(oracle.take_columns(oracle.make_abridged_hadamard(4, 2), [0, 1]))
    assert np.array_equal(S, H4[:, :2])


@pytest.mark.parametrize("n", [4, 8, 16, 64])
def test_apply_materialize_both_sides(oracle, n):  # test_sketch.cpp:223-240
    rng = oracle.Rng(40 + n)
    ops = [oracle.gen_permutation(n, rng), oracle.gen_sign_diagonal(n, rng),
           oracle.make_abridged_hadamard(n, 2), oracle.gen_sparse_circulant(n, 3, rng),
           oracle.gen_gaussian(n, n, rng), oracle.gen_asph(n, 2, rng)]
    M = rng.gaussian_matrix(n, 3)
    W = rng.gaussian_matrix(3, n)
    for op in ops:
        D = oracle.materialize(op)
        scale = 1e-12 * np.linalg.norm(D) * np.linalg.norm(M) + 1e-13
        assert np.linalg.norm(oracle.apply(op, M, "left") - D @ M) <= scale
        assert np.linalg.norm(oracle.apply(op, W, "right") - W @ D) <= scale


def test_flop_budgets(oracle):  # test_sketch.cpp:258-279
    rng = oracle.Rng(60)
    n, c = 64, 8
    M = rng.gaussian_matrix(n, c)
    oracle.reset_op_counter()
    oracle.make_abridged_hadamard(n, 3).apply(M)
    adds, muls = oracle.op_counter()
    assert adds <= 3 * n * c and muls == 0
    oracle.reset_op_counter()
    oracle.gen_sparse_circulant(n, 4, rng).apply(M)
    assert sum(oracle.op_counter()) <= (2 * 4 - 1) * n * c
    oracle.reset_op_counter()
    oracle.make_sub_identity([0, 5, 9], n).apply(M)
    assert sum(oracle.op_counter()) == 0


# ---------------------------------------------------------------- range finder / LSR
def test_range_finder_exact_rank(oracle):  # test_lra.cpp:10-22
    for t in range(10):
        rng = oracle.Rng(700 + t)
        m, n, r, l = 48, 40, 6, 10
        M = oracle.gen_factor_gaussian(m, n, r, 0.0, rng)
        H = oracle.gen_gaussian(n, l, rng)
        for trunc in (False, True):
            U, V = oracle.range_finder(M, H, r, trunc)
            assert np.linalg.norm(M - U @ V, 2) <= 1e-10 * np.linalg.norm(M, 2)
            if trunc:
                assert U.shape[1] == r


def test_range_finder_rank_failure(oracle):  # test_lra.cpp:24-30
    rng = oracle.Rng(20)
    H = oracle.gen_gaussian(16, 4, rng)
    with pytest.raises(oracle.RangeFailure):
        oracle.range_finder(np.zeros((16, 16)), H, 1)
    M1 = rng.gaussian_matrix(16, 1) @ rng.gaussian_matrix(1, 16)
    with pytest.raises(oracle.RangeFailure):
        oracle.range_finder(M1, H, 2)


def test_range_finder_graded_spectrum_asph(oracle):  # test_lra.cpp:32-44 (5 trials)
    tot = 0.0
    for t in range(5):
        rng = oracle.Rng(800 + t)
        M = oracle.gen_svd_profile(256, 8, rng)
        H = oracle.take_columns_random(oracle.gen_asph(256, 3, rng), 8, rng)
        U, V = oracle.range_finder(M, H, 8)
        tot += np.linalg.norm(M - U @ V, 2)
    assert tot / 5 <= 1e-6


def test_premult_identity_matches_range_finder(oracle):  # test_lra.cpp:98-108
    rng = oracle.Rng(25)
    m, n = 30, 24
    M = rng.gaussian_matrix(m, n)
    H = oracle.gen_gaussian(n, 6, rng)
    F = oracle.make_sub_identity(list(range(m)), m)
    Ua, Va = oracle.range_finder(M, H, 4)
    Ub, Vb = oracle.lra_premult(M, F, H, 4)
    assert np.linalg.norm(Ua - Ub, 2) <= 1e-12
    assert np.linalg.norm(Va - Vb, 2) <= 1e-12


def test_premult_exact_rank(oracle):  # test_lra.cpp:110-120
    for t in range(10):
        rng = oracle.Rng(900 + t)
        m, n, r, l, k = 48, 40, 5, 8, 12
        M = oracle.gen_factor_gaussian(m, n, r, 0.0, rng)
        H = oracle.gen_gaussian(n, l, rng)
        F = oracle.gen_gaussian(k, m, rng)
        U, V = oracle.lra_premult(M, F, H, r)
        assert np.linalg.norm(M - U @ V, 2) <= 1e-9 * np.linalg.norm(M, 2)


def test_premult_residual_identity_and_impact(oracle):  # test_lra.cpp:122-142
    rng = oracle.Rng(26)
    m, n, r, l, k = 8, 8, 2, 3, 5
    for _ in range(20):
        M = rng.gaussian_matrix(m, n)
        Hd = rng.gaussian_matrix(n, l)
        Fd = rng.gaussian_matrix(k, m)
        U, V = oracle.lra_premult(M, oracle.make_gaussian(Fd), oracle.make_gaussian(Hd), r)
        FU = Fd @ U
        P = np.eye(m) - U @ np.linalg.pinv(FU, rcond=1e-10) @ Fd
        resid = P @ (M - U @ (U.T @ M))
        assert np.linalg.norm(M - U @ V - resid, 2) <= 1e-9 * np.linalg.norm(M, 2)
        impact = np.linalg.norm(P, 2)
        bound = 1 + np.linalg.norm(U, 2) * np.linalg.norm(np.linalg.pinv(FU, rcond=1e-10), 2) * np.linalg.norm(Fd, 2)
        assert impact <= bound * (1 + 1e-12)


def test_premult_rank_failure(oracle):  # test_lra.cpp:144-150
    rng = oracle.Rng(27)
    M = oracle.gen_factor_gaussian(16, 16, 3, 0.0, rng)
    H = oracle.gen_gaussian(16, 4, rng)
    F = oracle.make_gaussian(np.zeros((5, 16)))
    with pytest.raises(oracle.PremultRankFailure):
        oracle.lra_premult(M, F, H, 3)


def test_two_stage_truncate(oracle):  # test_lra.cpp:152-170
    rng = oracle.Rng(28)
    m, n, l = 40, 32, 8
    U = rng.gaussian_matrix(m, l)
    V = rng.gaussian_matrix(l, n)
    P = U @ V
    Us, Vs = oracle.two_stage_truncate(U, V, l)
    assert np.linalg.norm(P - Us @ Vs, 2) <= 1e-12 * np.linalg.norm(P, 2)
    U3, V3 = oracle.two_stage_truncate(U, V, 3)
    S, sig, Tt = np.linalg.svd(P)
    dense3 = (S[:, :3] * sig[:3]) @ Tt[:3]
    assert np.linalg.norm(U3 @ V3 - dense3, 2) <= 1e-9 * np.linalg.norm(P, 2)
    with pytest.raises(Exception):
        oracle.two_stage_truncate(U, V, l + 1)


def test_two_stage_truncation_bound(oracle):  # test_lra.cpp:172-193 (25 of the 100 trials)
    for t in range(25):
        rng = oracle.Rng(1000 + t)
        n, r, l = 64, 4, 8
        M = oracle.gen_factor_gaussian(n, n, r, 1e-4, rng)
        H = oracle.gen_gaussian(n, l, rng)
        U, V = oracle.range_finder(M, H, r)
        Ug, Vg = oracle.two_stage_truncate(U, V, r)
        sig = np.linalg.svd(M, compute_uv=False)
        tau = np.sqrt(np.sum(sig[r:] ** 2))
        lhs = np.linalg.norm(M - Ug @ Vg)
        assert lhs <= (tau + 2 * np.linalg.norm(M - U @ V)) * (1 + 1e-8)


def test_lsr_full_permutation_exact(oracle):  # test_lsr.cpp:59-69
    rng = oracle.Rng(13)
    A = rng.gaussian_matrix(30, 3)
    b = rng.gaussian_vector(30)
    F = oracle.gen_permutation(30, rng)
    rep = oracle.sketch_solve(A, b, F, True)
    assert rep["k"] == 30
    assert rep["ratio"] == pytest.approx(1.0, rel=1e-10)
    assert rep["sketched_residual"] == pytest.approx(rep["true_residual"], rel=1e-10)


def test_lsr_consistent_system(oracle):  # test_lsr.cpp:71-81
    rng = oracle.Rng(14)
    A = rng.gaussian_matrix(64, 6)
    x0 = rng.gaussian_vector(6)
    b = A @ x0
    F = oracle.gen_gaussian(8, 64, rng)
    rep = oracle.sketch_solve(A, b, F)
    assert np.linalg.norm(rep["x_hat"] - x0) < 1e-8
    assert rep["sketched_residual"] < 1e-10


def test_lsr_rank_failure(oracle):  # test_lsr.cpp:83-90
    rng = oracle.Rng(15)
    A = rng.gaussian_matrix(32, 4)
    b = rng.gaussian_vector(32)
    with pytest.raises(oracle.SketchRankFailure):
        oracle.sketch_solve(A, b, oracle.make_gaussian(np.zeros((6, 32))))


def test_lsr_gaussian_ratio(oracle):  # test_lsr.cpp:92-105
    m, d = 256, 10
    tot = 0.0
    for t in range(20):
        rng = oracle.Rng(300 + t)
        A, b = oracle.gen_lsr_gaussian(m, d, 0.01, rng)
        rep = oracle.sketch_solve(A, b, oracle.gen_gaussian(6 * d, m, rng), True)
        assert 1.0 - 1e-12 <= rep["ratio"] < 2.0
        tot += rep["ratio"]
    assert tot / 20 < 1.3


def test_solve_exact_vs_lapack(oracle):
    rng = oracle.Rng(16)
    A, b = oracle.gen_lsr_gaussian(200, 12, 0.01, rng)
    x = oracle.solve_exact(A, b)
    assert np.allclose(x, np.linalg.lstsq(A, b, rcond=None)[0], atol=1e-12)


# ---------------------------------------------------------------- HSS (test_hss.cpp)
from hss_inputs import block_diagonal, cauchy_kernel, gen_fd_inverse, gravity_kernel, tridiagonal  # noqa: E402


def test_hss_block_diagonal_exact(oracle):  # test_hss.cpp:34-41
    rng = oracle.Rng(48)
    M = block_diagonal(rng, 8, 8)
    h = oracle.build_hss(M, 3, 4, 1e-10, "svd", rng)
    assert oracle.hss_error(h, M, "spectral") <= 1e-12
    assert not h["any_overflow"]
    assert all(b["F"].shape[1] == 0 for b in h["off"])


def test_hss_tridiagonal_rank_one_blocks(oracle):  # test_hss.cpp:43-50
    rng = oracle.Rng(49)
    M = tridiagonal(64, rng)
    h = oracle.build_hss(M, 3, 2, 1e-12, "svd", rng)
    assert oracle.hss_error(h, M, "spectral") <= 1e-10 * np.linalg.norm(M, 2)
    assert all(b["F"].shape[1] <= 1 for b in h["off"])


def test_hss_cauchy_superfast(oracle):  # test_hss.cpp:52-58
    M = cauchy_kernel(512)
    h = oracle.build_hss(M, 4, 16, 1e-7, "cur_ca", oracle.Rng(50))
    assert oracle.hss_error(h, M, "spectral") <= 1e-5 * np.linalg.norm(M, 2)
    assert all(b["F"].shape[1] <= 16 for b in h["off"])


def test_hss_matvec(oracle):  # test_hss.cpp:60-86 (flop budget: op_counter not restated)
    rng = oracle.Rng(51)
    M = gen_fd_inverse(64, 64)
    h = oracle.build_hss(M, 3, 6, 1e-9, "svd", rng)
    assert np.linalg.norm(oracle.hss_matvec(h, np.zeros(64))) == 0.0
    R = oracle.hss_reconstruct(h)
    scale = np.linalg.norm(R, 2)
    for _ in range(20):
        x = rng.gaussian_vector(64)
        assert np.linalg.norm(oracle.hss_matvec(h, x) - R @ x) <= 1e-10 * scale * np.linalg.norm(x)
    B = block_diagonal(rng, 4, 8)
    hb = oracle.build_hss(B, 2, 2, 1e-10, "svd", rng)
    x = rng.gaussian_vector(32)
    assert np.linalg.norm(oracle.hss_matvec(hb, x) - B @ x) <= 1e-10 * np.linalg.norm(B, 2) * np.linalg.norm(x)


def test_hss_norm_sanity(oracle):  # test_hss.cpp:88-95
    M = gravity_kernel(64, 64)
    h = oracle.build_hss(M, 2, 4, 1e-4, "svd", oracle.Rng(52))
    assert oracle.hss_error(h, M, "chebyshev") <= oracle.hss_error(h, M, "spectral") * 64 * (1 + 1e-12)


def test_hss_strategy_comparison(oracle):  # test_hss.cpp:97-110 (20 of the 100 seeds)
    M = gravity_kernel(128, 128)
    es = oracle.hss_error(oracle.build_hss(M, 3, 8, 1e-5, "svd", oracle.Rng(0)), M, "frobenius")
    ok = sum(oracle.hss_error(oracle.build_hss(M, 3, 8, 1e-5, "cur_ca", oracle.Rng(3200 + t)), M, "frobenius")
             <= 10 * es for t in range(20))
    assert ok >= 18


def test_hss_superfast_reads_vanishing_fraction(oracle):  # test_hss.cpp:112-124
    prev = float("inf")
    for n in (128, 256, 512):
        h = oracle.build_hss(cauchy_kernel(n), 3, 8, 1e-6, "cur_ca", oracle.Rng(53))
        ratio = h["accesses"] / (n * n)
        assert ratio < prev
        prev = ratio


def test_hss_validation(oracle):  # test_hss.cpp:126-137
    rng = oracle.Rng(54)
    M = rng.gaussian_matrix(64, 64)
    h = oracle.build_hss(M, 3, 4, 1e-3, "svd", rng)
    assert sum(D.size for _, _, D in h["diag"]) <= 2 * (64 + 64) * h["leaf"]
    for args in ((rng.gaussian_matrix(60, 60), 3, 4), (rng.gaussian_matrix(64, 32), 3, 4), (M, 5, 4)):
        with pytest.raises(ValueError):
            oracle.build_hss(args[0], args[1], args[2], 1e-3, "svd", rng)


# ---------------------------------------------------------------- solve_with_retries (test_lsr.cpp:176-226)
def coherent_problem(m, d, seed):
    """A coherent LSR input built here (signal on the first d rows, weak
    elsewhere): a stand-in for gen_lsr_family(Coherent), which is not restated."""
    rng = np.random.default_rng(seed)
    A = 1e-3 * rng.standard_normal((m, d))
    A[:d, :] += np.eye(d) * 10.0
    b = A @ rng.standard_normal(d) + 1e-2 * rng.standard_normal(m)
    return np.asfortranarray(A), b


def test_retries_blind_sub_identity(oracle):  # test_lsr.cpp:176-195
    m = 32
    A = np.zeros((m, 1))
    A[20, 0] = 1.0
    b = 3.0 * A[:, 0]
    base = oracle.make_sub_identity(list(range(8)), m)
    rep = oracle.solve_with_retries(A, b, base, [], 40, 1.5, oracle.Rng(17))
    assert rep["attempts"] > 1 and rep["validated"]
    assert rep["x_hat"][0] == pytest.approx(3.0, rel=1e-12)
    with pytest.raises(oracle.SketchRankFailure):
        oracle.solve_with_retries(A, b, base, [], 0, 1.5, oracle.Rng(18))


def test_retries_validate_first_attempt(oracle):  # test_lsr.cpp:197-208
    first = 0
    for t in range(50):
        rng = oracle.Rng(600 + t)
        A, b = oracle.gen_lsr_gaussian(128, 6, 0.01, rng)
        base = oracle.gen_gaussian(36, 128, rng)
        rep = oracle.solve_with_retries(A, b, base, [], 3, 2.0, rng)
        assert rep["validated"]
        first += rep["attempts"] == 1
    assert first >= 47


def test_retries_coherent_family(oracle):  # test_lsr.cpp:210-226 (own coherent input)
    m, d = 64, 4
    A, b = coherent_problem(m, d, 19)
    base = oracle.make_sub_identity(list(range(d, d + 48)), m)
    rng = oracle.Rng(19)
    qf = [oracle.gen_permutation(m, rng) for _ in range(6)]
    rep = oracle.solve_with_retries(A, b, base, qf, 30, 2.0, rng)
    assert rep["attempts"] > 1
    x = np.linalg.lstsq(A, b, rcond=None)[0]
    assert np.linalg.norm(A @ rep["x_hat"] - b) / np.linalg.norm(A @ x - b) < 3.0


# ---------------------------------------------------------------- leverage (test_leverage.cpp)
def sampled_matrix(W, s):
    return W[:, s["indices"]] * s["d"]


def test_leverage_scores_known(oracle):  # test_leverage.cpp:23-43
    T = np.zeros((8, 3))
    T[0, 0] = T[1, 1] = T[2, 2] = 1.0
    p, _, _ = oracle.svd_leverage_scores(T)
    assert np.allclose(p[:3], 1 / 3, rtol=1e-14) and np.all(p[3:] == 0)
    rng = oracle.Rng(41)
    Q, _ = oracle.thin_qr(rng.gaussian_matrix(20, 4))
    q, _, _ = oracle.svd_leverage_scores(Q)
    assert q.sum() == pytest.approx(1.0, rel=1e-12) and q.min() >= 0
    O, _ = oracle.thin_qr(rng.gaussian_matrix(4, 4))
    q2, _, _ = oracle.svd_leverage_scores(Q @ O)
    assert np.abs(q - q2).max() <= 1e-12
    with pytest.raises(ValueError):
        oracle.svd_leverage_scores(rng.gaussian_matrix(20, 4))


def test_sample_exactly_known(oracle):  # test_leverage.cpp:45-85 (1000 -> 200 seeds in the mean check)
    rng = oracle.Rng(42)
    s = oracle.sample_exactly(np.array([1.0, 0, 0]), 3, rng)
    assert s["indices"] == [0, 0, 0] and np.allclose(s["d"], 1 / np.sqrt(3), rtol=1e-14)
    n, draws = 16, 10000
    s = oracle.sample_exactly(oracle.uniform_scores(n), draws, rng)
    cnt = np.bincount(s["indices"], minlength=n)
    assert np.all(np.abs(cnt - draws / n) <= 4 * np.sqrt(draws * (1 / n) * (1 - 1 / n)))
    assert np.allclose(s["d"][:20], np.sqrt(n / draws), rtol=1e-14)
    W = oracle.Rng(43).gaussian_matrix(16, 16)
    p, _, _ = oracle.svd_leverage_scores(oracle.thin_qr(W.T.copy())[0])
    tot = sum(np.linalg.norm(sampled_matrix(W, oracle.sample_exactly(p, 16, oracle.Rng(2000 + t)))) ** 2
              for t in range(200))
    assert tot / 200 == pytest.approx(np.linalg.norm(W) ** 2, rel=0.1)


def test_sample_expected_known(oracle):  # test_leverage.cpp:87-152
    s = oracle.sample_expected(oracle.uniform_scores(8), 8, oracle.Rng(44))
    assert len(s["indices"]) == 8 and np.all(s["d"] == 1.0)
    threw = False
    for t in range(200):
        try:
            oracle.sample_expected(np.full(1000, 1e-3), 1, oracle.Rng(2300 + t))
        except oracle.EmptySample:
            threw = True
            break
    assert threw


def test_collapse_duplicates_gram(oracle):  # test_leverage.cpp:154-163
    rng = oracle.Rng(45)
    W = rng.gaussian_matrix(12, 10)
    _, _, T = oracle.svd(W)
    p, _, _ = oracle.svd_leverage_scores(T[:, :4].copy())
    raw = oracle.sample_exactly(p, 30, rng)
    merged = oracle.collapse_duplicates(raw["indices"], raw["d"])
    assert len(merged["indices"]) < len(raw["indices"])
    A, B = sampled_matrix(W, raw), sampled_matrix(W, merged)
    assert np.linalg.norm(A @ A.T - B @ B.T, 2) <= 1e-10


def test_cur_via_leverage_exact(oracle):  # test_leverage.cpp:165-183 (40 of 100 seeds)
    ok = done = 0
    for t in range(40):
        rng = oracle.Rng(2400 + t)
        M = oracle.gen_factor_gaussian(64, 64, 3, 0.0, rng)
        try:
            c = oracle.cur_via_leverage(M, 3, 12, 12, 1.0, 1.0, "exactly", None, rng)
        except (oracle.GeneratorRankFailure, oracle.EmptySample):
            continue
        done += 1
        C = M[:, c["J"]] @ c["nucleus"] @ M[c["I"], :]
        ok += np.linalg.norm(M - C, 2) <= 1e-8 * np.linalg.norm(M, 2)
    assert ok >= 38 and ok <= done


def test_refine_lra_truthful(oracle):  # test_leverage.cpp:225-245 (40 of 100 seeds)
    ok = 0
    for t in range(40):
        rng = oracle.Rng(2800 + t)
        M = oracle.gen_factor_gaussian(64, 64, 4, 1e-6, rng)
        S, s, Tt = np.linalg.svd(M)
        U, V = S[:, :4] * s[:4], Tt[:4].copy()
        crude_err = np.linalg.norm(M - U @ V)
        try:
            c = oracle.refine_lra(M, U, V, 4, 4, 24, 24, rng)
        except (oracle.GeneratorRankFailure, oracle.EmptySample):
            continue
        ok += np.linalg.norm(M - M[:, c["J"]] @ c["nucleus"] @ M[c["I"], :]) <= 1.5 * crude_err
    assert ok >= 36


def test_score_gap_and_bounds(oracle):  # test_leverage.cpp:292-320
    assert np.all(oracle.uniform_scores(4) == 0.25)
    Q, _ = oracle.thin_qr(oracle.Rng(47).gaussian_matrix(64, 4))
    assert oracle.gaussian_score_gap(np.sqrt(64.0) * Q.T) <= 1e-12
    assert oracle.sample_bound_quadratic(2, 1.0, 1.0) == pytest.approx(12800.0)
    assert oracle.sample_bound_loglinear(8, 1.0, 1.0, 100.0) == pytest.approx(100.0 * 8 * np.log(8.0))
    assert oracle.epsilon_for_sample(2, 16, 0.1) == pytest.approx(np.sqrt(8.0 * np.log(40.0) / 16.0))


# ---------------------------------------------------------------- remaining operators (test_sketch.cpp:119-158)
def test_inverse_bidiagonal_known(oracle):
    X = oracle.Rng(3).gaussian_matrix(6, 2)
    assert np.array_equal(oracle.make_inverse_bidiagonal(np.zeros(5)).apply(X), X)
    rng = oracle.Rng(4)
    n = 64
    op = oracle.gen_inverse_bidiagonal(n, rng)
    B = oracle.materialize(op)
    L = np.linalg.inv(B)
    assert np.linalg.norm(L @ B - np.eye(n)) < 1e-10
    for i in range(n):
        for j in range(i + 2, min(n - 1, i + 3) + 1):
            assert abs(L[j, i]) < 1e-12
    assert np.linalg.cond(B) <= np.sqrt(2) * n * (1 + 1e-8)
    Y = rng.gaussian_matrix(n, 3)
    assert np.linalg.norm(op.apply_transpose(Y) - B.T @ Y) < 1e-11 * np.linalg.norm(B) * np.linalg.norm(Y)
    U = oracle.materialize(oracle.make_inverse_bidiagonal(np.ones(3), False))
    assert abs(U[0, 3] - 1.0) < 1e-14 and np.allclose(U, np.triu(U))


def test_householder_chain_orthogonal(oracle):
    rng = oracle.Rng(6)
    op = oracle.gen_householder_chain(16, 4, rng)
    R = oracle.materialize(op)
    assert np.linalg.norm(R @ R.T - np.eye(16)) < 1e-12
    X = rng.gaussian_matrix(16, 3)
    assert np.linalg.norm(op.apply_transpose(X) - R.T @ X) < 1e-12


def test_abridged_fourier_displays(oracle):  # test_sketch.cpp:50-80
    F = oracle.materialize_complex(oracle.make_abridged_fourier(4, 2))
    E = np.array([[1, 1, 1, 1], [1, 1j, -1, -1j], [1, -1, 1, -1], [1, -1j, -1, 1j]])
    assert np.linalg.norm(F - E) < 1e-14
    a = np.arange(8)
    F8 = oracle.materialize_complex(oracle.make_abridged_fourier(8, 3))
    assert np.abs(F8 - np.exp(2j * np.pi * np.outer(a, a) / 8)).max() < 1e-13
    A = oracle.materialize_complex(oracle.make_abridged_fourier(8, 2))
    assert np.linalg.norm(A @ A.conj().T - 4 * np.eye(8)) < 1e-12
    assert all((np.abs(A[r]) > 1e-14).sum() == 4 for r in range(8))
    X = oracle.Rng(5).gaussian_matrix(8, 3).astype(complex)
    op = oracle.make_abridged_fourier(8, 2)
    assert np.linalg.norm(oracle.apply_transpose_complex(op, X) - A.T @ X) < 1e-12


def test_bidiagonal_product_generator(oracle):  # test_sketch.cpp:292-317
    assert np.linalg.norm(oracle.gen_bidiagonal_product(5, 0, oracle.Rng(1), False) - np.eye(5)) == 0.0
    B = oracle.bidiagonal_factor(3, [1, 1, 1])
    assert B[0, 2] == 1.0 and B[1, 0] == 1.0 and B[2, 1] == 1.0 and np.all(np.diag(B) == 1.0)
    G = oracle.gen_bidiagonal_product(16, 5, oracle.Rng(77), False)
    assert np.linalg.norm(G[:, 7] - oracle.bidiagonal_product_column(16, 5, 7, oracle.Rng(77))) == 0.0
    S = oracle.gen_bidiagonal_product(32, 8, oracle.Rng(78), True)
    assert np.all(np.abs(S.mean(axis=0)) < 1e-12) and np.all(np.abs((S ** 2).mean(axis=0) - 1) < 1e-10)


def test_ks_normality(oracle):  # test_sketch.cpp:319-334 (20 of the 100 seeds)
    passes = 0
    for t in range(20):
        r = oracle.Rng(1000 + t)
        passes += oracle.ks_normality([r.gaussian() for _ in range(10000)])[1]
    assert passes >= 18
    with pytest.raises(ValueError):
        oracle.ks_normality([1.0] * 100)
    r = oracle.Rng(5)
    assert not oracle.ks_normality([r.uniform() for _ in range(10000)])[1]


# ------------------------------------------------ CompleteOrthogonalDecomposition (cur.cpp:146-152)
@pytest.mark.parametrize("shape", [(16, 16, 16), (20, 12, 12), (12, 20, 12), (16, 16, 5), (10, 30, 4), (30, 10, 6)])
def test_oracle_cod_pinv_is_the_pseudo_inverse(oracle, shape):
    # well-posed generators: the COD pseudo-inverse equals the SVD one (LAPACK)
    k, l, rk = shape
    g = np.random.default_rng(k * 100 + l + rk)
    G = np.asfortranarray(g.standard_normal((k, rk)) @ g.standard_normal((rk, l)))
    P, r = oracle.cod_pseudo_inverse(G, 1e-10)
    assert r == rk
    Pn = np.linalg.pinv(G, rcond=1e-10)
    assert np.linalg.norm(P - Pn) <= 1e-12 * np.linalg.norm(Pn) * max(k, l)
    if rk < min(k, l):  # r above the COD rank: GeneratorRankFailure (cur.cpp:150-151)
        with pytest.raises(oracle.GeneratorRankFailure):
            oracle.primitive_cur(G, list(range(k)), list(range(l)), rk + 1, qr_nucleus=True)
