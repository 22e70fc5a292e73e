"""Leverage-score CUR (leverage.cpp:12-196) on the B200
against the oracle (needs a GPU: `-m gpu`). Same Rng seed -> same draws over
score vectors that agree to rounding -> the same index sets (asserted
exactly), nuclei within 1e-10 relative to the product's scale. Properties
restate test_leverage.cpp."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slra():
    import paper_1611_01391_b200 as s
    return s


def cur_err(M, c):
    return np.linalg.norm(M - M[:, c["J"]] @ c["nucleus"] @ M[c["I"], :])


def test_scores_vs_oracle(slra, oracle):
    rng = oracle.Rng(41)
    for shape in ((20, 4), (300, 8), (5000, 48)):
        Q, _ = oracle.thin_qr(rng.gaussian_matrix(*shape))
        p, _, r = slra.svd_leverage_scores(Q)
        po, _, _ = oracle.svd_leverage_scores(Q)
        assert r == shape[1] and np.allclose(p, po, rtol=1e-13, atol=1e-18)
    with pytest.raises(ValueError):
        slra.svd_leverage_scores(rng.gaussian_matrix(20, 4))


def test_sampling_matches_oracle(slra, oracle):
    p = np.abs(oracle.Rng(5).gaussian_vector(300))
    p /= p.sum()
    for l in (1, 17, 400):
        a = slra.sample_exactly(p, l, slra.Rng(l))
        b = oracle.sample_exactly(p, l, oracle.Rng(l))
        assert a["indices"] == b["indices"] and np.array_equal(a["d"], b["d"])
        a = slra.sample_expected(p, l, slra.Rng(l))
        b = oracle.sample_expected(p, l, oracle.Rng(l))
        assert a["indices"] == b["indices"] and np.array_equal(a["d"], b["d"])
        c = slra.collapse_duplicates(a["indices"], a["d"])
        d = oracle.collapse_duplicates(b["indices"], b["d"])
        assert c["indices"] == d["indices"] and np.array_equal(c["d"], d["d"])


@pytest.mark.parametrize("mode", ["exactly", "expected"])
@pytest.mark.parametrize("plain", [False, True])
@pytest.mark.parametrize("n,r,k", [(64, 3, 12), (256, 8, 64), (96, 4, 16)])
def test_cur_via_leverage_parity(slra, oracle, mode, plain, n, r, k):
    seed = 2400 + n + r + (mode == "expected") + 2 * plain
    M = oracle.gen_factor_gaussian(n, n, r, 1e-7, oracle.Rng(seed))
    try:
        co = oracle.cur_via_leverage(M, r, k, k, 1.0, 1.0, mode, None, oracle.Rng(seed + 1), plain)
    except (oracle.GeneratorRankFailure, oracle.EmptySample) as e:
        with pytest.raises((slra.GeneratorRankFailure, slra.EmptySample)):
            slra.cur_via_leverage(M, r, k, k, 1.0, 1.0, mode, None, slra.Rng(seed + 1), plain)
        return
    c = slra.cur_via_leverage(M, r, k, k, 1.0, 1.0, mode, None, slra.Rng(seed + 1), plain)
    assert c["I"] == co["I"] and c["J"] == co["J"]
    Cp = M[:, c["J"]] @ c["nucleus"] @ M[c["I"], :]
    Co = M[:, co["J"]] @ co["nucleus"] @ M[co["I"], :]
    assert np.linalg.norm(Cp - Co) <= 1e-9 * np.linalg.norm(M)


def test_cur_via_leverage_exact(slra):  # test_leverage.cpp:165-183 (all 100 seeds)
    ok = done = 0
    for t in range(100):
        rng = slra.Rng(2400 + t)
        M = slra.gen_factor_gaussian(64, 64, 3, 0.0, rng)
        try:
            c = slra.cur_via_leverage(M, 3, 12, 12, 1.0, 1.0, "exactly", None, rng)
        except (slra.GeneratorRankFailure, slra.EmptySample):
            continue
        done += 1
        C = M[:, c["J"]] @ c["nucleus"] @ M[c["I"], :]
        ok += np.linalg.norm(M - C, 2) <= 1e-8 * np.linalg.norm(M, 2)
    assert ok >= 95 and ok <= done


def test_uniform_scores_incoherent(slra):  # test_leverage.cpp:185-200
    tot = 0.0
    for t in range(20):
        rng = slra.Rng(2500 + t)
        M = slra.gen_factor_gaussian(256, 256, 8, 1e-6, rng)
        c = slra.cur_via_leverage(M, 8, 64, 64, 1.0, 1.0, "exactly", slra.uniform_scores(256), rng)
        tot += np.linalg.norm(M - M[:, c["J"]] @ c["nucleus"] @ M[c["I"], :], 2) / np.linalg.norm(M, 2)
        assert c["accesses"] <= 64 * 256 + 64 * 256 + 64 * 64
    assert tot / 20 <= 1e-3


def test_plain_vs_rescaled(slra):  # test_leverage.cpp:202-223
    ok = 0
    for t in range(50):
        M = slra.gen_factor_gaussian(96, 96, 4, 1e-7, slra.Rng(2600 + t))
        try:
            a = slra.cur_via_leverage(M, 4, 16, 16, 1.0, 1.0, "exactly", None, slra.Rng(2700 + t))
            b = slra.cur_via_leverage(M, 4, 16, 16, 1.0, 1.0, "exactly", None, slra.Rng(2700 + t), True)
        except (slra.GeneratorRankFailure, slra.EmptySample):
            continue
        ea, eb = cur_err(M, a), cur_err(M, b)
        ok += eb <= 10 * ea + 1e-12 and ea <= 10 * eb + 1e-12
    assert ok >= 45


def test_refine_lra(slra, oracle):  # test_leverage.cpp:225-263
    ok = crashes = 0
    for t in range(100):
        rng = slra.Rng(2800 + t)
        M = slra.gen_factor_gaussian(64, 64, 4, 1e-6, rng)
        S, s, Tt = np.linalg.svd(M)
        U, V = S[:, :4] * s[:4], Tt[:4].copy()
        try:
            c = slra.refine_lra(M, U, V, 4, 4, 24, 24, rng)
        except (slra.GeneratorRankFailure, slra.EmptySample):
            crashes += 1
            continue
        ok += cur_err(M, c) <= 1.5 * np.linalg.norm(M - U @ V)
    assert ok >= 90 and crashes <= 5
    # parity of the top-SVD step and one refinement
    rng = oracle.Rng(46)
    U, V = rng.gaussian_matrix(300, 6), rng.gaussian_matrix(6, 200)
    S, sig, T = slra.lra_to_top_svd(U, V, 4)
    So, sigo, To = oracle.lra_to_top_svd(U, V, 4)
    assert np.allclose(sig, sigo, rtol=1e-12) and np.allclose(S, So, atol=1e-10) and np.allclose(T, To, atol=1e-10)
    M = U @ V
    c = slra.refine_lra(M, U, V, 6, 4, 16, 16, slra.Rng(7))
    co = oracle.refine_lra(M, U, V, 6, 4, 16, 16, oracle.Rng(7))
    assert c["I"] == co["I"] and c["J"] == co["J"]


def test_score_gap(slra, oracle):  # test_leverage.cpp:292-310
    Q, _ = oracle.thin_qr(oracle.Rng(47).gaussian_matrix(64, 4))
    assert slra.gaussian_score_gap(np.sqrt(64.0) * Q.T) <= 1e-12
    ok = 0
    for t in range(100):
        G = slra.Rng(3000 + t).gaussian_matrix(8, 8192)
        g = slra.gaussian_score_gap(G)
        if t < 3:
            assert g == pytest.approx(oracle.gaussian_score_gap(G), rel=1e-9, abs=1e-15)
        ok += g <= 0.02 / 8
    assert ok >= 90
