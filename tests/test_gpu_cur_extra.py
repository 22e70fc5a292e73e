"""The remaining public entry points around the CUR / LRA path on the B200
against the oracle (needs a GPU: `-m gpu`): truncate_rank, condition_number,
cynical_cur, lra_to_top_svd(A, W, B), top_svd_to_cur (both selectors),
deterministic_error_diagnostic, posterior_error_estimate, and cur_evaluate in
the spectral / Chebyshev norms (cur.cpp:76-323, linalg.cpp:100-161,
lra.cpp:65-127)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def slra():
    import paper_1611_01391_b200 as s
    return s


def prod(M, c):
    return M[:, c["J"]] @ c["nucleus"] @ M[c["I"], :]


def test_truncate_rank_and_condition_number(slra, oracle):
    A = oracle.gen_factor_gaussian(120, 80, 6, 1e-9, oracle.Rng(1))
    U, V = slra.truncate_rank(A, 6)
    Uo, Vo = oracle.truncate_rank(A, 6)
    assert np.linalg.norm(U @ V - Uo @ Vo) <= TOL * np.linalg.norm(A)
    with pytest.raises(ValueError):
        slra.truncate_rank(A, 81)
    for D in (np.diag([4.0, 2.0, 1e-12]), np.diag([4.0, 2.0, 1e-9]), oracle.Rng(2).gaussian_matrix(30, 20)):
        assert slra.condition_number(D) == pytest.approx(oracle.condition_number(D), rel=1e-10)
    with pytest.raises(ValueError):
        slra.condition_number(np.zeros((3, 3)))


@pytest.mark.parametrize("seed", range(4))
def test_cynical_cur(slra, oracle, seed):
    M = oracle.gen_factor_gaussian(200, 160, 5, 1e-9, oracle.Rng(10 + seed))
    c = slra.cynical_cur(M, 40, 40, 10, 10, 5, slra.Rng(seed))
    co = oracle.cynical_cur(M, 40, 40, 10, 10, 5, oracle.Rng(seed))
    assert c["I"] == co["I"] and c["J"] == co["J"]
    assert np.linalg.norm(prod(M, c) - prod(M, co)) <= TOL * np.linalg.norm(M)
    with pytest.raises(ValueError):
        slra.cynical_cur(M, 40, 40, 50, 10, 5, slra.Rng(seed))


def test_lra_to_top_svd_general(slra, oracle):
    rng = oracle.Rng(3)
    A, W, B = rng.gaussian_matrix(300, 8), rng.gaussian_matrix(8, 6), rng.gaussian_matrix(6, 200)
    S, sig, T = slra.lra_to_top_svd3(A, W, B, 5)
    So, sigo, To = oracle.lra_to_top_svd3(A, W, B, 5)
    assert np.allclose(sig, sigo, rtol=1e-12)
    assert np.allclose(S, So, atol=1e-10) and np.allclose(T, To, atol=1e-10)


@pytest.mark.parametrize("sel", ["deterministic", "sampled"])
def test_top_svd_to_cur(slra, oracle, sel):
    M = oracle.gen_factor_gaussian(150, 120, 4, 0.0, oracle.Rng(4))
    S, s, Tt = np.linalg.svd(M)
    args = (np.ascontiguousarray(S[:, :4]), s[:4], np.ascontiguousarray(Tt[:4].T), 8, 8, 1.1, sel)
    c = slra.top_svd_to_cur(*args, slra.Rng(5))
    co = oracle.top_svd_to_cur(*args, oracle.Rng(5))
    assert c["I"] == co["I"] and c["J"] == co["J"]
    assert np.linalg.norm(c["nucleus"] - co["nucleus"]) <= 1e-9 * np.linalg.norm(co["nucleus"])
    assert np.linalg.norm(M - prod(M, c)) <= 1e-9 * np.linalg.norm(M)


def test_deterministic_error_diagnostic(slra, oracle):
    M = oracle.gen_factor_gaussian(96, 80, 6, 1e-5, oracle.Rng(6))
    b, a = slra.deterministic_error_diagnostic(M, slra.gen_gaussian(80, 12, slra.Rng(7)), 6)
    bo, ao = oracle.deterministic_error_diagnostic(M, oracle.gen_gaussian(80, 12, oracle.Rng(7)), 6)
    assert b == pytest.approx(bo, rel=1e-8) and a == pytest.approx(ao, rel=1e-8)
    assert a <= b * (1 + 1e-8)
    with pytest.raises(ValueError):
        slra.deterministic_error_diagnostic(np.zeros((600, 600)), slra.gen_gaussian(600, 4, slra.Rng(1)), 2)


def test_posterior_error_estimate(slra, oracle):
    M = oracle.gen_factor_gaussian(400, 300, 8, 1e-3, oracle.Rng(8))
    U, V = np.linalg.svd(M)[0][:, :8] * np.linalg.svd(M)[1][:8], np.linalg.svd(M)[2][:8]
    for q, s in ((20, 20), (5, 5), (1, 2)):
        e = slra.posterior_error_estimate(M, U, V, q, s, slra.Rng(q))
        eo = oracle.posterior_error_estimate(M, U, V, q, s, oracle.Rng(q))
        assert e[3] == eo[3]
        assert np.allclose(e[:3], eo[:3], rtol=1e-9)
    with pytest.raises(ValueError):
        slra.posterior_error_estimate(M, U, V, 1, 1, slra.Rng(0))


@pytest.mark.parametrize("norm", ["spectral", "chebyshev", "frobenius"])
def test_cur_evaluate_norms(slra, oracle, norm):
    M = oracle.gen_factor_gaussian(180, 140, 6, 1e-6, oracle.Rng(9))
    co = oracle.cross_approx(M, 6, 8, 8, [], 2, 1.1, None, oracle.Rng(9))
    co = co[0] if isinstance(co, tuple) else co
    v = slra.cur_evaluate(M, co["I"], co["J"], co["nucleus"], norm)
    vo = oracle.cur_evaluate(M, co["I"], co["J"], co["nucleus"], norm)
    assert v == pytest.approx(vo, rel=1e-7)
