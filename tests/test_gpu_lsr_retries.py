"""solve_with_retries (lsr.cpp:69-113) on the B200
against the oracle (needs a GPU: `-m gpu`): same Rng seeds give the same
re-randomised sketches, so attempts / validated flags must agree exactly and
x_hat within 1e-10 relative. Properties restate test_lsr.cpp:176-226."""
import numpy as np
import pytest

from test_oracle_pins import coherent_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slra():
    import paper_1611_01391_b200 as s
    return s


def same_report(rp, ro, scale=1.0):
    assert rp["attempts"] == ro["attempts"] and rp["validated"] == ro["validated"] and rp["k"] == ro["k"]
    assert np.linalg.norm(rp["x_hat"] - ro["x_hat"]) <= 1e-10 * max(scale, np.linalg.norm(ro["x_hat"]))


def test_retries_blind_sub_identity(slra, oracle):  # test_lsr.cpp:176-195
    m = 32
    A = np.zeros((m, 1))
    A[20, 0] = 1.0
    b = 3.0 * A[:, 0]
    rp = slra.solve_with_retries(A, b, slra.make_sub_identity(list(range(8)), m), [], 40, 1.5, slra.Rng(17))
    ro = oracle.solve_with_retries(A, b, oracle.make_sub_identity(list(range(8)), m), [], 40, 1.5, oracle.Rng(17))
    assert rp["attempts"] > 1 and rp["validated"] and rp["x_hat"][0] == pytest.approx(3.0, rel=1e-12)
    same_report(rp, ro)
    with pytest.raises(slra.SketchRankFailure):
        slra.solve_with_retries(A, b, slra.make_sub_identity(list(range(8)), m), [], 0, 1.5, slra.Rng(18))


def test_retries_validate_first_attempt(slra, oracle):  # test_lsr.cpp:197-208
    first = 0
    for t in range(50):
        rp_, ro_ = slra.Rng(600 + t), oracle.Rng(600 + t)
        A, b = slra.gen_lsr_gaussian(128, 6, 0.01, rp_)
        Ao, bo = oracle.gen_lsr_gaussian(128, 6, 0.01, ro_)
        assert np.array_equal(A, Ao) and np.array_equal(b, bo)
        rp = slra.solve_with_retries(A, b, slra.gen_gaussian(36, 128, rp_), [], 3, 2.0, rp_)
        ro = oracle.solve_with_retries(A, b, oracle.gen_gaussian(36, 128, ro_), [], 3, 2.0, ro_)
        assert rp["validated"]
        same_report(rp, ro)
        first += rp["attempts"] == 1
    assert first >= 47


def test_retries_coherent_family(slra, oracle):  # test_lsr.cpp:210-226 (own coherent input)
    m, d = 64, 4
    A, b = coherent_problem(m, d, 19)
    rp_, ro_ = slra.Rng(19), oracle.Rng(19)
    qp = [slra.gen_permutation(m, rp_) for _ in range(6)]
    qo = [oracle.gen_permutation(m, ro_) for _ in range(6)]
    rp = slra.solve_with_retries(A, b, slra.make_sub_identity(list(range(d, d + 48)), m), qp, 30, 2.0, rp_)
    ro = oracle.solve_with_retries(A, b, oracle.make_sub_identity(list(range(d, d + 48)), m), qo, 30, 2.0, ro_)
    assert rp["attempts"] > 1
    x = np.linalg.lstsq(A, b, rcond=None)[0]
    assert np.linalg.norm(A @ rp["x_hat"] - b) / np.linalg.norm(A @ x - b) < 3.0
    same_report(rp, ro)


@pytest.mark.parametrize("m,d,k", [(1 << 14, 64, 512), (1 << 16, 128, 2048)])
def test_retries_config4_style(slra, oracle, m, d, k):
    """CLI 'circulant' recipe at reduced size: validated on the first try."""
    rp_, ro_ = slra.Rng(m + d), oracle.Rng(m + d)
    A, b = oracle.gen_lsr_gaussian(m, d, 1e-6, oracle.Rng(7))
    sp, so = rp_.distinct_indices(k, m), ro_.distinct_indices(k, m)
    Fp = slra.make_product([slra.make_sub_identity(sp, m), slra.gen_sparse_circulant(m, 2, rp_),
                            slra.gen_sign_diagonal(m, rp_)])
    Fo = oracle.make_product([oracle.make_sub_identity(so, m), oracle.gen_sparse_circulant(m, 2, ro_),
                              oracle.gen_sign_diagonal(m, ro_)])
    rp = slra.solve_with_retries(A, b, Fp, [], 2, 2.0, rp_)
    ro = oracle.solve_with_retries(A, b, Fo, [], 2, 2.0, ro_)
    assert rp["validated"] and rp["attempts"] == 1
    same_report(rp, ro)
