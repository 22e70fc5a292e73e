"""The non-plan sketch operators of SURVEY.md §8f row 3 (sketch.cpp:286-383):
inverse bidiagonal (device scan) and the permuted Householder chain (device
GEMMs + row gathers), alone and inside composites, against the oracle
(needs a GPU: `-m gpu`). Properties restate test_sketch.cpp:119-158, 200-240."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slra():
    import paper_1611_01391_b200 as s
    return s


@pytest.mark.parametrize("n,c", [(2, 1), (64, 3), (1000, 7), (5000, 40), (1 << 16, 3)])
def test_inverse_bidiagonal_bit_exact(slra, oracle, n, c):
    rp, ro = slra.Rng(n), oracle.Rng(n)
    op, oo = slra.gen_inverse_bidiagonal(n, rp), oracle.gen_inverse_bidiagonal(n, ro)
    X = oracle.Rng(n + 1).gaussian_matrix(n, c)
    assert np.array_equal(op.apply(X), oo.apply(X))  # b = +-1: every step exact in both
    assert np.array_equal(op.apply_transpose(X), oo.apply_transpose(X))
    b = oracle.Rng(n + 2).gaussian_vector(n - 1) if n > 1 else np.zeros(0)
    for lower in (True, False):
        u, uo = slra.make_inverse_bidiagonal(b, lower), oracle.make_inverse_bidiagonal(b, lower)
        ref = uo.apply(X)
        assert np.linalg.norm(u.apply(X) - ref) <= 1e-13 * max(1.0, np.linalg.norm(ref))


@pytest.mark.parametrize("n,q,c", [(16, 4, 3), (256, 3, 5), (4096, 5, 2)])
def test_householder_chain_vs_oracle(slra, oracle, n, q, c):
    op = slra.gen_householder_chain(n, q, slra.Rng(6 + n))
    oo = oracle.gen_householder_chain(n, q, oracle.Rng(6 + n))
    X = oracle.Rng(7).gaussian_matrix(n, c)
    for f, g in ((op.apply, oo.apply), (op.apply_transpose, oo.apply_transpose)):
        assert np.linalg.norm(f(X) - g(X)) <= 1e-13 * np.linalg.norm(X)
    if n <= 256:
        R = slra.materialize(op)
        assert np.linalg.norm(R @ R.T - np.eye(n)) < 1e-12


def test_known_properties(slra):  # test_sketch.cpp:119-158
    X = slra.Rng(3).gaussian_matrix(6, 2)
    assert np.array_equal(slra.make_inverse_bidiagonal(np.zeros(5)).apply(X), X)
    rng = slra.Rng(4)
    n = 64
    op = slra.gen_inverse_bidiagonal(n, rng)
    B = slra.materialize(op)
    L = np.linalg.inv(B)
    assert np.linalg.norm(L @ B - np.eye(n)) < 1e-10
    assert all(abs(L[j, i]) < 1e-12 for i in range(n) for j in range(i + 2, min(n - 1, i + 3) + 1))
    assert np.linalg.cond(B) <= np.sqrt(2) * n * (1 + 1e-8)
    Y = rng.gaussian_matrix(n, 3)
    assert np.linalg.norm(op.apply_transpose(Y) - B.T @ Y) < 1e-11 * np.linalg.norm(B) * np.linalg.norm(Y)
    U = slra.materialize(slra.make_inverse_bidiagonal(np.ones(3), False))
    assert abs(U[0, 3] - 1.0) < 1e-14 and np.allclose(U, np.triu(U))


@pytest.mark.parametrize("n", [4, 8, 16, 64])
def test_apply_both_sides_and_slices(slra, oracle, n):  # test_sketch.cpp:200-240
    rp, ro = slra.Rng(40 + n), oracle.Rng(40 + n)
    ops = [(slra.gen_inverse_bidiagonal(n, rp), oracle.gen_inverse_bidiagonal(n, ro)),
           (slra.gen_householder_chain(n, 3, rp), oracle.gen_householder_chain(n, 3, ro))]
    M = oracle.Rng(1).gaussian_matrix(n, 3)
    W = oracle.Rng(2).gaussian_matrix(3, n)
    for op, oo in ops:
        D = slra.materialize(op)
        sc = 1e-12 * np.linalg.norm(D) * np.linalg.norm(M) + 1e-13
        assert np.linalg.norm(slra.apply(op, M, "left") - D @ M) <= sc
        assert np.linalg.norm(slra.apply(op, W, "right") - W @ D) <= sc
        assert np.linalg.norm(slra.apply(op, W, "right") - oracle.apply(oo, W, "right")) <= sc
        sl, so = slra.take_columns_random(op, n // 2, rp), oracle.take_columns_random(oo, n // 2, ro)
        Ds, Dso = slra.materialize(sl), oracle.materialize(so)
        assert np.linalg.norm(Ds - Dso) <= 1e-12 * np.linalg.norm(Dso)
        assert np.linalg.cond(Ds) <= np.linalg.cond(D) * (1 + 1e-8)


def test_sketch_solve_through_non_plan_operators(slra, oracle):
    """F = SubIdentity(k of m) . HouseholderChain: the sketched system is
    formed by the device application, then solved as usual."""
    m, d, k = 2048, 16, 256
    A, b = oracle.gen_lsr_gaussian(m, d, 1e-6, oracle.Rng(5))
    rp, ro = slra.Rng(8), oracle.Rng(8)
    sp, so = rp.distinct_indices(k, m), ro.distinct_indices(k, m)
    Fp = slra.make_product([slra.make_sub_identity(sp, m), slra.gen_householder_chain(m, 2, rp)])
    Fo = oracle.make_product([oracle.make_sub_identity(so, m), oracle.gen_householder_chain(m, 2, ro)])
    rep = slra.sketch_solve(A, b, Fp, False)
    ref = oracle.sketch_solve(A, b, Fo, False)
    assert np.linalg.norm(rep["x_hat"] - ref["x_hat"]) <= 1e-10 * np.linalg.norm(ref["x_hat"])
    assert rep["sketched_residual"] == pytest.approx(ref["sketched_residual"], rel=1e-8)
    # the inverse-bidiagonal preconditioner on its own (k = m)
    Fb = slra.gen_inverse_bidiagonal(m, slra.Rng(9))
    Fbo = oracle.gen_inverse_bidiagonal(m, oracle.Rng(9))
    rep = slra.sketch_solve(A, b, Fb, False)
    ref = oracle.sketch_solve(A, b, Fbo, False)
    assert np.linalg.norm(rep["x_hat"] - ref["x_hat"]) <= 1e-9 * np.linalg.norm(ref["x_hat"])


def test_abridged_fourier_displays(slra):  # test_sketch.cpp:50-80
    F = slra.materialize_complex(slra.make_abridged_fourier(4, 2))
    E = np.array([[1, 1, 1, 1], [1, 1j, -1, -1j], [1, -1, 1, -1], [1, -1j, -1, 1j]])
    assert np.linalg.norm(F - E) < 1e-14
    a = np.arange(8)
    F8 = slra.materialize_complex(slra.make_abridged_fourier(8, 3))
    assert np.abs(F8 - np.exp(2j * np.pi * np.outer(a, a) / 8)).max() < 1e-13
    A = slra.materialize_complex(slra.make_abridged_fourier(8, 2))
    assert np.linalg.norm(A @ A.conj().T - 4 * np.eye(8)) < 1e-12
    assert all((np.abs(A[r]) > 1e-14).sum() == 4 for r in range(8))
    X = slra.Rng(5).gaussian_matrix(8, 3).astype(complex)
    op = slra.make_abridged_fourier(8, 2)
    assert np.linalg.norm(slra.apply_transpose_complex(op, X) - A.T @ X) < 1e-12
    with pytest.raises(RuntimeError):
        op.apply(np.eye(8))  # complex operator: real application refused (std::logic_error)


@pytest.mark.parametrize("n,d,c", [(8, 2, 3), (64, 6, 5), (4096, 3, 7), (1024, 10, 2), (96, 5, 4)])
def test_abridged_fourier_bit_exact(slra, oracle, n, d, c):
    rng = oracle.Rng(n + d)
    X = rng.gaussian_matrix(n, c) + 1j * rng.gaussian_matrix(n, c)
    op, oo = slra.make_abridged_fourier(n, d), oracle.make_abridged_fourier(n, d)
    assert np.array_equal(slra.apply_complex(op, X), oracle.apply_complex(oo, X))
    assert np.array_equal(slra.apply_transpose_complex(op, X), oracle.apply_transpose_complex(oo, X))


def test_complex_products(slra, oracle):
    """A real operator acts on both planes; products chain complex factors
    (sketch.cpp:26-37, 511-540)."""
    n = 256
    rp, ro = slra.Rng(3), oracle.Rng(3)
    sp, so = rp.distinct_indices(32, n), ro.distinct_indices(32, n)
    Fp = slra.make_product([slra.make_sub_identity(sp, n), slra.make_abridged_fourier(n, 3), slra.gen_sign_diagonal(n, rp)])
    Fo = oracle.make_product([oracle.make_sub_identity(so, n), oracle.make_abridged_fourier(n, 3),
                              oracle.gen_sign_diagonal(n, ro)])
    X = oracle.Rng(4).gaussian_matrix(n, 3) + 0j
    assert np.array_equal(slra.apply_complex(Fp, X), oracle.apply_complex(Fo, X))
    Y = oracle.Rng(5).gaussian_matrix(32, 2) + 1j * oracle.Rng(6).gaussian_matrix(32, 2)
    assert np.array_equal(slra.apply_transpose_complex(Fp, Y), oracle.apply_transpose_complex(Fo, Y))


def test_sum_operator(slra, oracle):
    """Signed sums (sketch.cpp:446-500): device applications accumulated in
    the reference's order; alone, in products, transposed and complex."""
    n = 128
    rp, ro = slra.Rng(21), oracle.Rng(21)
    Sp = slra.make_sum([slra.gen_sparse_circulant(n, 3, rp), slra.gen_asph(n, 2, rp, True),
                        slra.gen_householder_chain(n, 2, rp)], [1, -1, 1])
    So = oracle.make_sum([oracle.gen_sparse_circulant(n, 3, ro), oracle.gen_asph(n, 2, ro, True),
                          oracle.gen_householder_chain(n, 2, ro)], [1, -1, 1])
    X = oracle.Rng(2).gaussian_matrix(n, 4)
    for f, g in ((Sp.apply, So.apply), (Sp.apply_transpose, So.apply_transpose)):
        assert np.linalg.norm(f(X) - g(X)) <= 1e-13 * np.linalg.norm(g(X))
    sel = list(range(0, n, 4))
    Fp = slra.make_product([slra.make_sub_identity(sel, n), Sp])
    Fo = oracle.make_product([oracle.make_sub_identity(sel, n), So])
    assert np.linalg.norm(Fp.apply(X) - Fo.apply(X)) <= 1e-13 * np.linalg.norm(Fo.apply(X))
    Z = X + 1j * oracle.Rng(3).gaussian_matrix(n, 4)
    Cp = slra.make_sum([slra.make_abridged_fourier(n, 3), slra.gen_sign_diagonal(n, slra.Rng(4))], [1, -1])
    Co = oracle.make_sum([oracle.make_abridged_fourier(n, 3), oracle.gen_sign_diagonal(n, oracle.Rng(4))], [1, -1])
    assert np.array_equal(slra.apply_complex(Cp, Z), oracle.apply_complex(Co, Z))
    with pytest.raises(ValueError):
        slra.make_sum([slra.gen_sign_diagonal(n, rp), slra.gen_sign_diagonal(n, rp)], [1, 2])


def test_generators_match_oracle(slra, oracle):
    assert np.array_equal(slra.gen_bidiagonal_product(64, 6, slra.Rng(9), True),
                          oracle.gen_bidiagonal_product(64, 6, oracle.Rng(9), True))
    assert np.array_equal(slra.bidiagonal_product_column(64, 6, 5, slra.Rng(9)),
                          oracle.bidiagonal_product_column(64, 6, 5, oracle.Rng(9)))
    x = [slra.Rng(3).gaussian() for _ in range(1)]
    r = slra.Rng(1000)
    sample = [r.gaussian() for _ in range(10000)]
    assert slra.ks_normality(sample) == oracle.ks_normality(sample)
    X = oracle.Rng(1).gaussian_matrix(64, 3)
    Dp, Do = slra.gen_scaled_diagonal(64, slra.Rng(2)), oracle.gen_scaled_diagonal(64, oracle.Rng(2))
    assert np.array_equal(Dp.apply(X), Do.apply(X))
