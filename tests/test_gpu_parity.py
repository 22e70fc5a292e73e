"""Parity of the B200 path against the CPU oracle (needs a GPU: `-m gpu`).

Every call goes through the product: paper_1611_01391_b200 (C++ host layer)
-> include/slra_cuda.h C-ABI -> sm_100a kernels. The oracle (oracle/) is the
checker. Tolerances follow BASELINE.json north_star: index sets bit-exact
where well-posed, sketches bit-exact, factors/residuals within 1e-10
relative to ||A||_F.
"""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

TOL = 1e-10


@pytest.fixture(scope="module")
def slra():
    import paper_1611_01391_b200 as s
    return s


# ---------------------------------------------------------------- sketches (bit-exact)
@pytest.mark.parametrize("n,l,s", [(64, 8, 3), (512, 48, 4), (4096, 48, 4)])
def test_sparse_circulant_right_bit_exact(slra, oracle, n, l, s):
    seed = 100 + n
    rp, ro = slra.Rng(seed), oracle.Rng(seed)
    Hp = slra.take_columns_random(slra.gen_sparse_circulant(n, s, rp), l, rp)
    Ho = oracle.take_columns_random(oracle.gen_sparse_circulant(n, s, ro), l, ro)
    M = oracle.Rng(seed + 1).gaussian_matrix(257, n)
    assert np.array_equal(slra.apply(Hp, M, "right"), oracle.apply(Ho, M, "right"))


@pytest.mark.parametrize("n,l,d", [(16, 8, 2), (512, 48, 3), (4096, 48, 3), (1024, 32, 4)])
def test_asph_right_bit_exact(slra, oracle, n, l, d):
    seed = 200 + n + d
    rp, ro = slra.Rng(seed), oracle.Rng(seed)
    Hp = slra.take_columns_random(slra.gen_asph(n, d, rp), l, rp)
    Ho = oracle.take_columns_random(oracle.gen_asph(n, d, ro), l, ro)
    M = oracle.Rng(seed + 1).gaussian_matrix(300, n)
    assert np.array_equal(slra.apply(Hp, M, "right"), oracle.apply(Ho, M, "right"))


@pytest.mark.parametrize("m,k,s", [(1024, 64, 2), (1 << 14, 512, 2)])
def test_lsr_sketch_rows_bit_exact(slra, oracle, m, k, s):
    # CLI "circulant" recipe: Product{SubIdentity(k of m), Z_f(s), D}
    seed = 300 + m
    rp, ro = slra.Rng(seed), oracle.Rng(seed)
    sel_p, sel_o = rp.distinct_indices(k, m), ro.distinct_indices(k, m)
    Fp = slra.make_product([slra.make_sub_identity(sel_p, m), slra.gen_sparse_circulant(m, s, rp),
                            slra.gen_sign_diagonal(m, rp)])
    Fo = oracle.make_product([oracle.make_sub_identity(sel_o, m), oracle.gen_sparse_circulant(m, s, ro),
                              oracle.gen_sign_diagonal(m, ro)])
    W = oracle.Rng(seed + 1).gaussian_matrix(m, 9)
    assert np.array_equal(Fp.apply(W), Fo.apply(W))
    U = slra.make_sub_identity(sel_p, m)
    assert np.array_equal(U.apply(W), W[sel_o, :])


def test_materialize_known_answers(slra):  # test_sketch.cpp:29-48
    H4 = np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]], float)
    E1 = np.array([[1, 0, 1, 0], [0, 1, 0, 1], [1, 0, -1, 0], [0, 1, 0, -1]], float)
    assert np.array_equal(slra.materialize(slra.make_abridged_hadamard(4, 1)), E1)
    assert np.array_equal(slra.materialize(slra.make_abridged_hadamard(4, 2)), H4)
    assert np.array_equal(slra.materialize(slra.make_abridged_hadamard(8, 3)), np.block([[H4, H4], [H4, -H4]]))


@pytest.mark.parametrize("n", [4, 8, 16, 64])
def test_apply_both_sides_vs_oracle(slra, oracle, n):  # test_sketch.cpp:223-240
    seed = 40 + n
    rp, ro = slra.Rng(seed), oracle.Rng(seed)
    pairs = [(slra.gen_permutation(n, rp), oracle.gen_permutation(n, ro)),
             (slra.gen_sign_diagonal(n, rp), oracle.gen_sign_diagonal(n, ro)),
             (slra.make_abridged_hadamard(n, 2), oracle.make_abridged_hadamard(n, 2)),
             (slra.gen_sparse_circulant(n, 3, rp), oracle.gen_sparse_circulant(n, 3, ro)),
             (slra.gen_asph(n, 2, rp), oracle.gen_asph(n, 2, ro))]
    M = oracle.Rng(seed + 7).gaussian_matrix(n, 3)
    W = oracle.Rng(seed + 8).gaussian_matrix(3, n)
    for p, o in pairs:
        assert np.array_equal(slra.apply(p, M, "left"), oracle.apply(o, M, "left"))
        assert np.array_equal(slra.apply(p, W, "right"), oracle.apply(o, W, "right"))
        assert np.array_equal(p.apply_transpose(M), o.apply_transpose(M))


# ---------------------------------------------------------------- dense kernels
@pytest.mark.parametrize("m,c", [(2, 1), (8, 3), (256, 16), (300, 48), (4096, 48), (16384, 64), (5000, 33)])
def test_thin_qr_vs_oracle(slra, oracle, m, c):
    A = oracle.Rng(m + c).gaussian_matrix(m, c)
    Q, R = slra.thin_qr(A)
    Qo, Ro = oracle.thin_qr(A)
    assert (np.diag(R) >= 0).all()
    assert np.linalg.norm(Q.T @ Q - np.eye(c)) <= 1e-13 * c
    assert np.linalg.norm(Q @ R - A) <= 1e-13 * np.linalg.norm(A) * c
    assert np.allclose(Q, Qo, atol=1e-11) and np.allclose(R, Ro, atol=1e-11 * np.abs(Ro).max())


def test_thin_qr_known_answer(slra):  # test_linalg.cpp:45-52
    Q, R = slra.thin_qr(np.array([[3.0], [4.0]]))
    assert abs(Q[0, 0] - 0.6) < 1e-15 and abs(Q[1, 0] - 0.8) < 1e-15 and abs(R[0, 0] - 5) < 1e-14


def test_thin_qr_rank_deficient_tsqr(slra, oracle):
    # config-3 style strip: numerically rank ~6 of 64; Q must stay orthonormal
    m = 16384
    r = oracle.Rng(3)
    x = np.array([r.uniform() for _ in range(m)])
    y = 2 + np.array([r.uniform() for _ in range(64)])
    A = 1.0 / (x[:, None] - y[None, :])
    Q, R = slra.thin_qr(A)
    assert np.linalg.norm(Q.T @ Q - np.eye(64)) <= 1e-12
    assert np.linalg.norm(Q @ R - A) <= 1e-13 * np.linalg.norm(A) * 64


# every rows-per-lane instantiation of the Jacobi kernel (p = 1..64 -> RPG 1..8,
# odd RPG included) on the one-CTA, tall (QR + square Jacobi) and wide paths
@pytest.mark.parametrize("shape", [(2, 2), (7, 5), (5, 7), (64, 64), (32, 32), (256, 48), (4096, 48), (48, 300),
                                   (17, 9), (9, 17), (20, 20), (33, 33), (40, 23), (56, 50), (61, 61),
                                   (300, 20), (4096, 20), (1000, 33), (20, 700), (5000, 57)])
def test_svd_vs_oracle(slra, oracle, shape):
    A = oracle.Rng(sum(shape) + 5).gaussian_matrix(*shape)
    S, sig, T = slra.svd(A)
    So, sigo, To = oracle.svd(A)
    assert np.allclose(sig, sigo, rtol=1e-12, atol=1e-14 * sigo[0])
    p = min(shape)
    assert np.linalg.norm(S @ np.diag(sig) @ T.T - A) <= 1e-12 * np.linalg.norm(A) * p
    for j in range(S.shape[1]):  # sign rule (linalg.cpp:87-96)
        assert S[np.argmax(np.abs(S[:, j])), j] >= 0
    assert np.allclose(S, So, atol=1e-9) and np.allclose(T, To, atol=1e-9)


def test_numerical_rank_and_pinv(slra):
    D = np.diag([1.0, 1e-10])
    assert slra.numerical_rank(D, 1e-6) == 1 and slra.numerical_rank(D, 1e-11, True) == 2
    A = np.random.default_rng(0).standard_normal((5, 3))
    assert np.allclose(slra.pseudo_inverse(A), np.linalg.pinv(A), atol=1e-13)


@pytest.mark.parametrize("ta,tb,m,n,k", [(0, 0, 64, 64, 64), (1, 0, 32, 4096, 4096), (0, 1, 100, 37, 23),
                                         (1, 1, 7, 9, 130), (0, 0, 4096, 48, 48), (1, 0, 257, 257, 4096),
                                         # the stream-K skinny W^T B kernel: ragged n and K, r = 1 .. 56, fewer
                                         # stage units than CTAs, many column tiles over a short K, one tile
                                         # over a long K; odd K (unaligned: the generic kernel)
                                         (1, 0, 13, 1000, 1026), (1, 0, 56, 130, 4098), (1, 0, 1, 70, 256),
                                         (1, 0, 48, 5000, 300), (1, 0, 33, 64, 20000), (1, 0, 8, 3, 777)])
def test_gemm_vs_numpy(slra, ta, tb, m, n, k):
    import ctypes
    import torch
    from paper_1611_01391_b200 import capi
    lib = capi.load()
    ctx = ctypes.c_void_p()
    assert lib.slra_ctx_create(0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(ctx)) == 0
    g = torch.Generator().manual_seed(m * n + k)
    A = torch.randn((k, m) if ta else (m, k), dtype=torch.float64, generator=g)
    B = torch.randn((n, k) if tb else (k, n), dtype=torch.float64, generator=g)
    Af, Bf = A.t().contiguous().cuda(), B.t().contiguous().cuda()  # column-major storage
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda")
    st = lib.slra_gemm(ctx, ta, tb, m, n, k, 1.0, Af.data_ptr(), A.shape[0], Bf.data_ptr(), B.shape[0], 0.0,
                       C.data_ptr(), m)
    assert st == 0
    torch.cuda.synchronize()
    ref = (A.t() if ta else A) @ (B.t() if tb else B)
    assert torch.allclose(C.t().cpu(), ref, atol=1e-12 * k ** 0.5 * 4)
    # alpha != 1, and the same bits on a second call (fixed-order combines)
    C2 = torch.zeros_like(C)
    for out in (C, C2):
        assert lib.slra_gemm(ctx, ta, tb, m, n, k, ctypes.c_double(-2.5), Af.data_ptr(), A.shape[0], Bf.data_ptr(),
                             B.shape[0], ctypes.c_double(0.0), out.data_ptr(), m) == 0
    torch.cuda.synchronize()
    assert torch.allclose(C.t().cpu(), -2.5 * ref, atol=1e-12 * k ** 0.5 * 10)
    assert torch.equal(C, C2)
    lib.slra_ctx_destroy(ctx)


@pytest.mark.parametrize("m,n,inner", [(64, 64, 8), (100, 77, 5), (256, 256, 16), (1000, 130, 33),
                                       (4096, 4096, 32), (300, 200, 0), (129, 65, 70)])
def test_lowrank_residual_vs_numpy(slra, m, n, inner):
    import ctypes
    import torch
    from paper_1611_01391_b200 import capi
    lib = capi.load()
    ctx = ctypes.c_void_p()
    assert lib.slra_ctx_create(0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(ctx)) == 0
    g = torch.Generator().manual_seed(m + n + inner)
    A = torch.randn(n, m, dtype=torch.float64, generator=g)  # A^T row-major = A column-major
    P = torch.randn(max(inner, 1), m, dtype=torch.float64, generator=g)
    Q = torch.randn(n, max(inner, 1), dtype=torch.float64, generator=g)
    dA, dP, dQ = A.cuda(), P.cuda(), Q.cuda()
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    st = lib.slra_lowrank_residual(ctx, dA.data_ptr(), m, m, n, dP.data_ptr(), m, dQ.data_ptr(), max(inner, 1),
                                   inner, out.data_ptr())
    assert st == 0
    torch.cuda.synchronize()
    Am, Pm, Qm = A.t().numpy(), P.t().numpy()[:, :inner], Q.t().numpy()[:inner, :]
    rs = np.sum((Am - Pm @ Qm) ** 2)
    ns = np.sum(Am ** 2)
    o = out.cpu().numpy()
    assert abs(o[0] - rs) <= 1e-12 * max(rs, ns) and abs(o[1] - ns) <= 1e-12 * ns
    lib.slra_ctx_destroy(ctx)


# ---------------------------------------------------------------- maxvol / CUR
def test_maxvol_known_answers(slra):  # test_cur.cpp:16-33
    A = np.zeros((9, 3))
    A[0, 0] = A[1, 1] = A[2, 2] = 1.0
    assert set(slra.maxvol_rows(A)) >= {0, 1, 2}
    assert slra.maxvol_rows(np.array([[1.0], [2.0], [-3.0]]), 1.0) == [2]
    with pytest.raises(slra.SelectionFailure):
        slra.maxvol_rows(np.zeros((5, 2)))


@pytest.mark.parametrize("m,r,seed", [(64, 4, 31), (256, 16, 1), (256, 32, 2), (500, 20, 3)])
def test_maxvol_vs_oracle(slra, oracle, m, r, seed):
    A, _ = oracle.thin_qr(oracle.Rng(seed).gaussian_matrix(m, r))
    I = slra.maxvol_rows(A, 1.1)
    assert I == oracle.maxvol_rows(A, 1.1)
    B = A @ np.linalg.inv(A[I, :])
    assert np.abs(B).max() <= 1.1 * (1 + 1e-12)


@pytest.mark.parametrize("m,c,seed", [(256, 16, 5), (256, 32, 6), (200, 20, 7)])
def test_select_rows_spanning_vs_oracle(slra, oracle, m, c, seed):
    A = oracle.Rng(seed).gaussian_matrix(m, c)
    assert slra.select_rows_spanning(A, c) == oracle.select_rows_spanning(A, c)
    assert slra.select_rows_spanning(A, c - 3) == oracle.select_rows_spanning(A, c - 3)


def test_primitive_cur_known_answers(slra, oracle):  # test_cur.cpp:80-108
    M = np.diag([5.0, 4, 3, 2, 1, 0.5])
    c = slra.primitive_cur(M, [0, 1, 2], [0, 1, 2], 3)
    R = slra.cur_reconstruct(M, c["I"], c["J"], c["nucleus"])
    assert np.linalg.norm(R[:3, :3] - M[:3, :3]) <= 1e-12
    D = np.zeros((8, 8))
    D[5, 5] = 1.0
    with pytest.raises(slra.GeneratorRankFailure):
        slra.primitive_cur(D, [0, 1], [0, 1], 1)
    rng = oracle.Rng(32)
    M = oracle.gen_factor_gaussian(40, 30, 3, 0.0, rng)
    I, J = rng.distinct_indices(5, 40), rng.distinct_indices(4, 30)
    c = slra.primitive_cur(M, I, J, 3)
    assert c["accesses"] == 20
    co = oracle.primitive_cur(M, I, J, 3)
    nA = np.linalg.norm(M)
    assert np.linalg.norm(slra.cur_reconstruct(M, I, J, c["nucleus"]) -
                          oracle.cur_reconstruct(M, I, J, co["nucleus"])) <= TOL * nA


@pytest.mark.parametrize("seed", range(8))
def test_cross_approx_config1_parity(slra, oracle, seed):
    """Config 1: 256x256 factor-Gaussian + 1e-8 noise, r=8, k=l=16, 3 sweeps."""
    A = slra.gen_factor_gaussian(256, 256, 8, 1e-8, slra.Rng(seed))
    assert np.array_equal(A, oracle.gen_factor_gaussian(256, 256, 8, 1e-8, oracle.Rng(seed)))
    init = slra.Rng(1000 + seed).distinct_indices(16, 256)
    g = slra.cross_approx(A, 8, 16, 16, init, 3, 1.1, slra.Rng(0))
    o = oracle.cross_approx(A, 8, 16, 16, init, 3, 1.1, None, oracle.Rng(0))
    assert g["I"] == o["I"] and g["J"] == o["J"]
    for sg, so in zip(g["trace"], o["trace"]):
        assert sg["rows"] == so["rows"] and sg["cols"] == so["cols"]
        # |det Q[J,:]| of a strip whose trailing directions sit at the 1e-8
        # noise level: conditioning ~ eps * sigma_1 / sigma_16 ~ 1e-7
        assert abs(sg["volume_proxy"] - so["volume_proxy"]) <= 1e-5 * max(so["volume_proxy"], 1e-300)
    nA = np.linalg.norm(A)
    Cg = slra.cur_reconstruct(A, g["I"], g["J"], g["nucleus"])
    Co = oracle.cur_reconstruct(A, o["I"], o["J"], o["nucleus"])
    assert np.linalg.norm(Cg - Co) <= TOL * nA
    eg = slra.cur_evaluate(A, g["I"], g["J"], g["nucleus"])
    eo = oracle.cur_evaluate(A, o["I"], o["J"], o["nucleus"])
    assert abs(eg - eo) <= TOL * nA
    assert eg / nA < 1e-6
    assert g["accesses"] <= 3 * (16 * 256 + 256 * 16) + 16 * 16


def test_cross_approx_exact_rank(slra, oracle):  # test_cur.cpp:145-155
    rng = oracle.Rng(35)
    m, n, r = 64, 48, 5
    M = oracle.gen_factor_gaussian(m, n, r, 0.0, rng)
    init = rng.distinct_indices(r, m)
    c = slra.cross_approx(M, r, r, r, init, 1, 1.1, slra.Rng(0))
    err = np.linalg.norm(M - slra.cur_reconstruct(M, c["I"], c["J"], c["nucleus"]), 2)
    assert err <= 1e-9 * np.linalg.norm(M, 2)
    assert len(c["trace"]) == 2
    assert c["accesses"] <= r * n + m * r + 2 * r * r


# ------------------------------------------------ large strips (config 3 path)
@pytest.mark.parametrize("seed", range(3))
def test_cross_approx_large_well_posed(slra, oracle, seed):
    """Strips taller than one SM (TSQR + grid-wide maxvol) on a well-posed
    rank-64 input: ordered I,J and every trace step bit-exact vs the oracle."""
    m = n = 2048
    k = 64
    A = slra.gen_factor_gaussian(m, n, k, 1e-8, slra.Rng(seed))
    init = slra.Rng(500 + seed).distinct_indices(k, m)
    g = slra.cross_approx(A, 48, k, k, init, 2, 1.1, slra.Rng(0))
    o = oracle.cross_approx(A, 48, k, k, init, 2, 1.1, None, oracle.Rng(0))
    assert g["I"] == o["I"] and g["J"] == o["J"]
    for sg, so in zip(g["trace"], o["trace"]):
        assert sg["rows"] == so["rows"] and sg["cols"] == so["cols"]
        assert abs(sg["volume_proxy"] - so["volume_proxy"]) <= 1e-6 * abs(so["volume_proxy"])
    nA = np.linalg.norm(A)
    eg = slra.cur_evaluate(A, g["I"], g["J"], g["nucleus"])
    eo = oracle.cur_evaluate(A, o["I"], o["J"], o["nucleus"])
    assert abs(eg - eo) <= TOL * nA
    # factored nucleus (inner dimension r) gives the same residual
    p = slra.primitive_cur(A, g["I"], g["J"], 48)
    assert p["tsig"].shape == (k, 48) and p["sr"].shape == (k, 48)
    assert np.linalg.norm(p["tsig"] @ p["sr"].T - p["nucleus"]) <= 1e-12 * np.linalg.norm(p["nucleus"])
    ef = slra.cur_evaluate_factored(A, g["I"], g["J"], p["tsig"], p["sr"])
    assert abs(ef - eo) <= TOL * nA


def _cauchy_replay_check(slra, oracle, A, g, k):
    """Replay parity (SURVEY.md §7 hard part 1): the oracle's adaptive-rank
    nucleus and residual on the GPU's I,J."""
    I, J = g["I"], g["J"]
    G = A[np.ix_(I, J)]
    rk = oracle.numerical_rank(G, 1e-10, True)
    assert rk == g["r"]
    ro = oracle.primitive_cur(A, I, J, rk)
    eo = oracle.cur_evaluate(A, I, J, ro["nucleus"])
    nA = np.linalg.norm(A)
    cond = 64 * 2.2e-16 * np.linalg.norm(A[:, J]) * np.linalg.norm(ro["nucleus"], 2) * np.linalg.norm(A[I, :])
    tol = TOL * nA + cond
    p = slra.primitive_cur(A, I, J, 0)
    assert p["r"] == rk
    ef = slra.cur_evaluate_factored(A, I, J, p["tsig"], p["sr"])
    eu = slra.cur_evaluate(A, I, J, p["nucleus"])
    assert abs(ef - eo) <= tol and abs(eu - eo) <= tol
    return ef / nA


@pytest.mark.parametrize("n,seed", [(4096, 0), (4096, 1), (1024, 2)])
def test_cross_approx_cauchy_reduced(slra, oracle, n, seed):
    """Config 3 at reduced size: 1/(x-y) block, k=l=64, 5 sweeps, adaptive r."""
    k = 64
    A = slra.gen_cauchy_block(n, n, slra.Rng(seed))
    r = oracle.Rng(seed)
    x = np.array([r.uniform() for _ in range(n)])
    y = np.array([2.0 + r.uniform() for _ in range(n)])
    assert np.array_equal(A, 1.0 / (x[:, None] - y[None, :]))
    init = slra.Rng(700 + seed).distinct_indices(k, n)
    g = slra.cross_approx(A, 0, k, k, init, 5, 1.1, slra.Rng(0))
    o = oracle.cross_approx(A, 1, k, k, init, 5, 1.1, None, oracle.Rng(0))
    same = sum(sg["rows"] == so["rows"] and sg["cols"] == so["cols"] for sg, so in zip(g["trace"], o["trace"]))
    # pivots beyond the strip's eps-rank (~9) pick among rounding-noise
    # directions: the contract there is replay parity, not identical sets,
    # plus per half-sweep the selection spans the strip's well-determined
    # subspace as well as the oracle's maxvol does
    rel = _cauchy_replay_check(slra, oracle, A, g, k)
    assert rel < 1e-9
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_config5 import check_half_sweeps
    spans = check_half_sweeps(A, g["trace"], o["trace"])
    print(f"config-3 reduced n={n}: {same}/{len(o['trace'])} trace steps identical, rel err {rel:.2e}, "
          f"(rank, gpu, oracle) span coefficients {spans}")


def test_cross_approx_cauchy_full_config3(slra, oracle):
    """Config 3 at full size (16384^2): replay parity on the GPU's I,J."""
    n, k = 16384, 64
    A = slra.gen_cauchy_block(n, n, slra.Rng(3))
    init = slra.Rng(703).distinct_indices(k, n)
    g = slra.cross_approx(A, 0, k, k, init, 5, 1.1, slra.Rng(0))
    rel = _cauchy_replay_check(slra, oracle, A, g, k)
    assert rel < 1e-9
    o = oracle.cross_approx(A, 1, k, k, init, 5, 1.1, None, oracle.Rng(0))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_config5 import check_half_sweeps
    print(f"config-3 full: span coefficients per half-sweep {check_half_sweeps(A, g['trace'], o['trace'])}")


def _log_block(oracle, b, master=0, m=256):
    r = oracle.Rng(oracle.Rng.derive_seed(master, b))
    px = []
    for _ in range(m):
        px.append((r.uniform(), r.uniform()))
    qx = []
    for _ in range(m):
        qx.append((4.0 + r.uniform(), r.uniform()))
    P, Q = np.array(px), np.array(qx)
    dx = P[:, 0][:, None] - Q[:, 0][None, :]
    dy = P[:, 1][:, None] - Q[:, 1][None, :]
    return 0.5 * np.log(dx * dx + dy * dy), r


def test_log_kernel_generator_matches(slra, oracle):
    K, _ = _log_block(oracle, 3)
    Kp = slra.gen_log_kernel_block(256, 256, slra.Rng(slra.Rng.derive_seed(0, 3)))
    assert np.allclose(K, Kp, rtol=0, atol=1e-15)


def test_batched_config5_parity(slra, oracle):
    """Config 5 subset: 64 independent 256x256 log-kernel blocks, adaptive r<=16, k=l=32, 2 sweeps."""
    import torch
    nb, m, k = 64, 256, 32
    blocks, inits = [], []
    for b in range(nb):
        Kb = slra.gen_log_kernel_block(m, m, slra.Rng(slra.Rng.derive_seed(0, b)))
        blocks.append(Kb)
        inits.append(slra.Rng(slra.Rng.derive_seed(1, b)).distinct_indices(k, m))
    A = torch.from_numpy(np.stack([Kb.T for Kb in blocks])).cuda()  # each block column-major
    init = torch.tensor(inits, dtype=torch.int64, device="cuda")
    I = torch.zeros((nb, k), dtype=torch.int64, device="cuda")
    J = torch.zeros((nb, k), dtype=torch.int64, device="cuda")
    U = torch.zeros((nb, k * k), dtype=torch.float64, device="cuda")
    rr = torch.zeros(nb, dtype=torch.int64, device="cuda")
    status = torch.zeros(nb, dtype=torch.int32, device="cuda")
    rs = torch.zeros(nb, dtype=torch.float64, device="cuda")
    ns = torch.zeros(nb, dtype=torch.float64, device="cuda")
    slra.cross_approx_batched_device(A.data_ptr(), m, m * m, nb, m, m, 0, k, k, init.data_ptr(), 2, 1.1,
                                     I.data_ptr(), J.data_ptr(), U.data_ptr(), rr.data_ptr(), status.data_ptr(),
                                     rs.data_ptr(), ns.data_ptr())
    torch.cuda.synchronize()
    assert (status.cpu() == 0).all()
    exact_sets = 0
    for b in range(nb):
        Kb = blocks[b]
        o = oracle.cross_approx(Kb, 1, k, k, inits[b], 2, 1.1, None, oracle.Rng(0))
        Ib, Jb = I[b].tolist(), J[b].tolist()
        exact_sets += (Ib == o["I"] and Jb == o["J"])
        nK = np.linalg.norm(Kb)
        # replay parity: the oracle's nucleus on the GPU's I,J (adaptive rank)
        G = Kb[np.ix_(Ib, Jb)]
        rk = oracle.numerical_rank(G, 1e-10, True)
        assert rk == int(rr[b])
        ro = oracle.primitive_cur(Kb, Ib, Jb, rk)
        eo = oracle.cur_evaluate(Kb, Ib, Jb, ro["nucleus"])
        # r_eff sits at the 1e-10 cut, so C U R carries a rounding error of
        # order eps ||C|| ||U|| ||R||; the tolerance adds that conditioning
        # term to the north_star 1e-10 ||A||_F bound.
        Cm, Rm = Kb[:, Jb], Kb[Ib, :]
        cond = 64 * 2.2e-16 * np.linalg.norm(Cm) * np.linalg.norm(ro["nucleus"], 2) * np.linalg.norm(Rm)
        tol = TOL * nK + cond
        eg = np.sqrt(rs[b].item())
        assert eg <= eo + tol and abs(eg - eo) <= tol
        assert abs(np.sqrt(ns[b].item()) - nK) <= 1e-13 * nK
        Ug = U[b].cpu().numpy().reshape(k, k).T
        Cg = oracle.cur_reconstruct(Kb, Ib, Jb, Ug)
        Co = oracle.cur_reconstruct(Kb, Ib, Jb, ro["nucleus"])
        assert np.linalg.norm(Cg - Co) <= tol
    print(f"config-5 subset: {exact_sets}/{nb} blocks with index sets identical to the oracle")


# ---------------------------------------------------------------- range finder (config 2)
def _config2_matrix(n, seed, device_qr=True):
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    Gu = torch.randn(n, n, dtype=torch.float64, generator=g).cuda()
    Gv = torch.randn(n, n, dtype=torch.float64, generator=g).cuda()
    U, Ru = torch.linalg.qr(Gu)
    V, Rv = torch.linalg.qr(Gv)
    U = U * torch.sign(torch.diagonal(Ru))[None, :]
    V = V * torch.sign(torch.diagonal(Rv))[None, :]
    j = torch.arange(n, dtype=torch.float64, device="cuda")
    sig = torch.where(j < 32, 0.5 ** j, torch.full_like(j, 1e-12))
    return ((U * sig[None, :]) @ V.T).cpu().numpy()


@pytest.mark.parametrize("n", [1024, 4096])
@pytest.mark.parametrize("kind", ["circulant", "asph"])
def test_range_finder_config2_parity(slra, oracle, n, kind):
    A = _config2_matrix(n, 7 + n)
    seed = 77
    rp, ro = slra.Rng(seed), oracle.Rng(seed)
    if kind == "circulant":
        Hp = slra.take_columns_random(slra.gen_sparse_circulant(n, 4, rp), 48, rp)
        Ho = oracle.take_columns_random(oracle.gen_sparse_circulant(n, 4, ro), 48, ro)
    else:
        Hp = slra.take_columns_random(slra.gen_asph(n, 3, rp), 48, rp)
        Ho = oracle.take_columns_random(oracle.gen_asph(n, 3, ro), 48, ro)
    nA = np.linalg.norm(A)
    for trunc in (True, False):
        U, V = slra.range_finder(A, Hp, 32, trunc)
        Uo, Vo = oracle.range_finder(A, Ho, 32, trunc)
        assert U.shape == Uo.shape and V.shape == Vo.shape
        assert np.linalg.norm(U @ V - Uo @ Vo) <= TOL * nA
        if trunc:
            assert np.allclose(U, Uo, atol=1e-12), np.abs(U - Uo).max()
        err = np.linalg.norm(A - U @ V) / nA
        assert err < 1e-9


def test_range_finder_batched_host_matches_single(slra):
    """The e2e entry (one upload of A, both config-2 multipliers batched)
    returns what range_finder returns per multiplier."""
    import torch
    n = 1024
    A = _config2_matrix(n, 5)
    rp = slra.Rng(3)
    Hs = [slra.take_columns_random(slra.gen_sparse_circulant(n, 4, rp), 48, rp),
          slra.take_columns_random(slra.gen_asph(n, 3, rp), 48, rp)]
    host = torch.from_numpy(np.asfortranarray(A).T.copy().reshape(-1)).pin_memory()  # column-major bytes
    out = slra.range_finder_batched_host(host.data_ptr(), n, n, Hs, 32, True)
    nA = np.linalg.norm(A)
    for (U, V, rs, ns), H in zip(out, Hs):
        U1, V1 = slra.range_finder(A, H, 32, True)
        assert np.allclose(U, U1, atol=1e-13) and np.allclose(V, V1, atol=1e-13 * nA)
        assert abs(np.sqrt(rs) - np.linalg.norm(A - U1 @ V1)) <= 1e-12 * nA
        assert abs(np.sqrt(ns) - nA) <= 1e-13 * nA


@pytest.mark.parametrize("cluster", [True, False])
@pytest.mark.parametrize("m,n,l,r", [(1000, 300, 13, 9), (4096, 512, 48, 32), (1531, 200, 64, 40), (777, 200, 29, 17),
                                     (523, 200, 64, 40), (64, 64, 8, 5), (16384, 128, 48, 20),
                                     (40000, 96, 24, 12)])
def test_range_finder_cholqr_paths_vs_oracle(slra, oracle, monkeypatch, cluster, m, n, l, r):
    """The sketch's QR (shifted CholeskyQR3) on both of its paths — the fused
    8-CTA cluster kernel (the sketch resident in shared memory for the three
    passes) and the multi-kernel passes (SLRA_NO_CLUSTER_CHOLQR=1; also what
    shapes beyond the cluster's shared memory or too short to stage the R
    product take: the last four here) — against the oracle's Householder
    thin_qr pipeline, on ragged shapes: m not a multiple of 8, l not a multiple
    of 8, l = 64."""
    monkeypatch.setenv("SLRA_NO_CLUSTER_CHOLQR", "0" if cluster else "1")
    rg = np.random.default_rng(m + l)
    sig = np.where(np.arange(r + 3) < r, 0.6 ** np.arange(r + 3), 1e-12)
    A = (rg.standard_normal((m, r + 3)) * sig) @ rg.standard_normal((r + 3, n))
    rp, ro = slra.Rng(5), oracle.Rng(5)
    Hp = slra.take_columns_random(slra.gen_sparse_circulant(n, 4, rp), l, rp)
    Ho = oracle.take_columns_random(oracle.gen_sparse_circulant(n, 4, ro), l, ro)
    nA = np.linalg.norm(A)
    for trunc in (True, False):
        U, V = slra.range_finder(A, Hp, r, trunc)
        Uo, Vo = oracle.range_finder(A, Ho, r, trunc)
        assert U.shape == Uo.shape and V.shape == Vo.shape
        assert np.linalg.norm(U @ V - Uo @ Vo) <= TOL * nA
        if not trunc:  # BasisQr: U is the thin Q itself
            assert np.linalg.norm(U.T @ U - np.eye(U.shape[1])) <= 1e-13 * np.sqrt(l) * 8


def test_range_finder_rank_failure(slra):  # test_lra.cpp:24-30
    rng = slra.Rng(20)
    H = slra.take_columns_random(slra.gen_sparse_circulant(64, 3, rng), 8, rng)
    with pytest.raises(slra.RangeFailure):
        slra.range_finder(np.zeros((64, 64)), H, 1)


# ---------------------------------------------------------------- LSR (config 4, reduced)
@pytest.mark.parametrize("kind", ["uniform", "sparse"])
def test_sketch_solve_config4_reduced(slra, oracle, kind):
    m, d, k = 1 << 15, 256, 4096
    A, b = slra.gen_lsr_gaussian(m, d, 1e-6, slra.Rng(9))
    Ao, bo = oracle.gen_lsr_gaussian(m, d, 1e-6, oracle.Rng(9))
    assert np.array_equal(A, Ao) and np.array_equal(b, bo)
    rp, ro = slra.Rng(10), oracle.Rng(10)
    if kind == "uniform":
        Fp = slra.make_sub_identity(rp.distinct_indices(k, m), m)
        Fo = oracle.make_sub_identity(ro.distinct_indices(k, m), m)
    else:
        sp, so = rp.distinct_indices(k, m), ro.distinct_indices(k, m)
        Fp = slra.make_product([slra.make_sub_identity(sp, m), slra.gen_sparse_circulant(m, 2, rp),
                                slra.gen_sign_diagonal(m, rp)])
        Fo = oracle.make_product([oracle.make_sub_identity(so, m), oracle.gen_sparse_circulant(m, 2, ro),
                                  oracle.gen_sign_diagonal(m, ro)])
    g = slra.sketch_solve(A, b, Fp, False)
    o = oracle.sketch_solve(A, b, Fo, False)
    xo = o["x_hat"]
    assert np.linalg.norm(g["x_hat"] - xo) <= 1e-10 * np.linalg.norm(xo)
    assert abs(g["sketched_residual"] - o["sketched_residual"]) <= 1e-8 * o["sketched_residual"]
    rg = slra.residual_norm(A, b, g["x_hat"])
    ro_ = oracle.residual_norm(A, b, xo)
    assert abs(rg - ro_) <= 1e-10 * np.linalg.norm(b)


def test_sketch_solve_known_answers(slra):  # test_lsr.cpp:59-90
    rng = slra.Rng(13)
    A = rng.gaussian_matrix(30, 3)
    b = rng.gaussian_vector(30)
    F = slra.gen_permutation(30, rng)
    rep = slra.sketch_solve(A, b, F, True)
    assert rep["k"] == 30 and abs(rep["ratio"] - 1.0) <= 1e-10
    rng = slra.Rng(15)
    A = rng.gaussian_matrix(32, 4)
    b = rng.gaussian_vector(32)
    Z = slra.make_product([slra.make_sub_identity([0, 1, 2, 3, 4, 5], 32), slra.make_sign_diagonal(np.ones(32))])
    with pytest.raises(slra.SketchRankFailure):
        slra.sketch_solve(np.zeros((32, 4)) + 0.0, b, Z)


# ---------------------------------------------------------------- C-A early stop (a15)
@pytest.mark.parametrize("seed,tol", [(0, 1e-3), (1, 0.0), (2, 1e-6)])
def test_cross_approx_stop_tol_parity(slra, oracle, seed, tol):
    """cross_approx with stop_tol (cur.cpp:235-249): the posterior estimate
    (lra.cpp:88-127, 20 x 20 sampled entries) after every horizontal
    half-sweep; same trace length, index sets, estimates and Rng stream."""
    A = slra.gen_factor_gaussian(256, 256, 8, 1e-8, slra.Rng(40 + seed))
    nA = np.linalg.norm(A)
    init = slra.Rng(60 + seed).distinct_indices(16, 256)
    rg, ro = slra.Rng(7), oracle.Rng(7)
    g = slra.cross_approx(A, 8, 16, 16, init, 4, 1.1, rg, tol * nA)
    o = oracle.cross_approx(A, 8, 16, 16, init, 4, 1.1, tol * nA, ro)
    assert len(g["trace"]) == len(o["trace"])
    assert g["I"] == o["I"] and g["J"] == o["J"]
    for sg, so in zip(g["trace"], o["trace"]):
        assert sg["rows"] == so["rows"] and sg["cols"] == so["cols"]
        if so["error_estimate"] is None:
            assert sg["error_estimate"] is None
        else:
            assert abs(sg["error_estimate"] - so["error_estimate"]) <= 1e-6 * so["error_estimate"] + 1e-12 * nA
    assert rg.next_u64() == ro.next_u64()  # the caller's stream advanced identically
    if tol > 0:
        assert len(o["trace"]) < 8  # stopped early


def test_cross_approx_stop_tol_probe_failure(slra, oracle):
    """r above the generator rank: every probe fails (no estimate, no draws)
    and the final primitive_cur raises GeneratorRankFailure, as the reference."""
    A = slra.gen_factor_gaussian(128, 128, 5, 0.0, slra.Rng(3))
    init = slra.Rng(4).distinct_indices(12, 128)
    with pytest.raises(slra.GeneratorRankFailure):
        slra.cross_approx(A, 8, 12, 12, init, 2, 1.1, slra.Rng(0), 1e-3)
    with pytest.raises(oracle.GeneratorRankFailure):
        oracle.cross_approx(A, 8, 12, 12, init, 2, 1.1, 1e-3, oracle.Rng(0))


# ---------------------------------------------------------------- edge cases
def test_select_rows_spanning_padding_branch(slra, oracle):  # cur.cpp:125-134
    A = oracle.Rng(41).gaussian_matrix(200, 10)
    for count in (10, 13, 17):
        assert slra.select_rows_spanning(A, count) == oracle.select_rows_spanning(A, count)


@pytest.mark.parametrize("m,c,seed", [(3000, 24, 1), (9000, 64, 2)])
def test_tall_selection_grid_path(slra, oracle, m, c, seed):
    """Strips taller than one SM: maxvol_rows and select_rows_spanning run the
    grid-wide cooperative kernel (select: after TSQR)."""
    A = oracle.Rng(seed).gaussian_matrix(m, c)
    assert slra.select_rows_spanning(A, c) == oracle.select_rows_spanning(A, c)
    Q, _ = oracle.thin_qr(A)
    I = slra.maxvol_rows(Q, 1.1)
    assert I == oracle.maxvol_rows(Q, 1.1)
    B = Q @ np.linalg.inv(Q[I, :])
    assert np.abs(B).max() <= 1.1 * (1 + 1e-12)


def test_invalid_arguments_raise(slra):  # std::invalid_argument in the reference
    A = slra.Rng(1).gaussian_matrix(40, 30)
    with pytest.raises(ValueError):
        slra.maxvol_rows(A[:, :5], 0.9)  # h < 1 (cur.cpp:91)
    with pytest.raises(ValueError):
        slra.maxvol_rows(A[:3, :5])  # m < r (cur.cpp:90)
    with pytest.raises(ValueError):
        slra.select_rows_spanning(A, 41)  # count > rows (cur.cpp:120)
    with pytest.raises(ValueError):
        slra.primitive_cur(A, [0, 1], [0, 1, 2], 3)  # |I| < r (cur.cpp:139-140)
    with pytest.raises(ValueError):
        slra.cross_approx(A, 5, 4, 6, [], 1, 1.1, slra.Rng(0))  # k < r (cur.cpp:205-206)
    rp = slra.Rng(2)
    H = slra.take_columns_random(slra.gen_sparse_circulant(30, 2, rp), 8, rp)
    with pytest.raises(ValueError):
        slra.range_finder(A, H, 9, True)  # r > l


def test_rank_deficient_lsr_raises(slra):  # lsr.cpp:52-55
    rng = slra.Rng(17)
    A = rng.gaussian_matrix(200, 6)
    A[:, 5] = A[:, 4]  # exactly dependent columns
    b = rng.gaussian_vector(200)
    F = slra.make_sub_identity(rng.distinct_indices(64, 200), 200)
    with pytest.raises(slra.SketchRankFailure):
        slra.sketch_solve(A, b, F, False)


def test_residual_ragged_and_empty_inner(slra):
    import torch
    rng = np.random.default_rng(5)
    for m, n, inner in [(129, 33, 0), (257, 95, 7), (64, 31, 2)]:
        A = rng.standard_normal((m, n))
        P = rng.standard_normal((m, max(inner, 1)))[:, :inner]
        Q = rng.standard_normal((max(inner, 1), n))[:inner, :]
        ref = np.linalg.norm(A - P @ Q) ** 2 if inner else np.linalg.norm(A) ** 2
        At = torch.from_numpy(np.asfortranarray(A).T.copy()).cuda()
        Pt = torch.from_numpy(np.asfortranarray(P).T.copy()).cuda() if inner else At
        Qt = torch.from_numpy(np.asfortranarray(Q).T.copy()).cuda() if inner else At
        out = torch.zeros(2, dtype=torch.float64, device="cuda")
        slra.lowrank_residual_device(At.data_ptr(), m, m, n, Pt.data_ptr(), m, Qt.data_ptr(), max(inner, 1), inner,
                                     out.data_ptr())
        o = out.cpu().numpy()
        assert abs(o[0] - ref) <= 1e-12 * max(ref, 1.0) and abs(o[1] - np.linalg.norm(A) ** 2) <= 1e-12 * o[1]


# ---------------------------------------------------------------- no silent fallback
def test_native_library_loaded(slra):
    import os
    maps = open("/proc/self/maps").read()
    assert "libslra_cuda.so" in maps and "libslra.so" in maps
    assert slra.launch_count() > 0
    assert os.path.dirname(slra.__file__) in maps


def test_integration_glue_cross_approx_on_gpu(slra, oracle, tmp_path):
    """the reference-side dispatch (tests/integration/,
    linked against libslra_cuda.so only) on the config-1 problem returns the
    oracle's ordered I, J."""
    import subprocess
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_host_cpu import build_integration_example, write_integration_input
    exe = build_integration_example(tmp_path)
    A = slra.gen_factor_gaussian(256, 256, 8, 1e-8, slra.Rng(5))
    init = slra.Rng(1005).distinct_indices(16, 256)
    inp = str(tmp_path / "in.bin")
    write_integration_input(inp, A, init, 3, 8)
    p = subprocess.run([exe, inp], capture_output=True, text=True)
    assert p.returncode == 0, p.stdout + p.stderr
    lines = dict(line.split(" ", 1) for line in p.stdout.strip().splitlines())
    o = oracle.cross_approx(A, 8, 16, 16, init, 3, 1.1, None, oracle.Rng(0))
    assert [int(v) for v in lines["I"].split()] == o["I"]
    assert [int(v) for v in lines["J"].split()] == o["J"]
    assert int(lines["r"]) == 8 and int(lines["steps"]) == 6


@pytest.mark.parametrize("n,k,loops", [(4096, 64, 2), (200, 16, 3)])
def test_cauchy_function_oracle_bit_identical(n, k, loops):
    """Config 3's block as a FunctionOracle (slra_cross_approx_cauchy +
    slra_cur_residual_factored_cauchy, oracle.hpp:43-54): strips, generator
    and the residual pass evaluate 1/(x_i - y_j) instead of reading the
    materialised matrix — the same selections, nucleus factors and residual
    bits as the dense entry points."""
    import torch
    import paper_1611_01391_b200 as slra
    rng = slra.Rng(123)
    x = torch.tensor([rng.uniform() for _ in range(n)], dtype=torch.float64, device="cuda")
    y = torch.tensor([2.0 + rng.uniform() for _ in range(n)], dtype=torch.float64, device="cuda")
    At = (1.0 / (x[None, :] - y[:, None])).contiguous()  # column-major A: At[j, i] = A(i, j)
    init = torch.tensor(slra.Rng(7).distinct_indices(k, n), dtype=torch.int64, device="cuda")

    def bufs():
        return dict(I=torch.zeros(k, dtype=torch.int64, device="cuda"), J=torch.zeros(k, dtype=torch.int64,
                                                                                       device="cuda"),
                    U=torch.zeros(k * k, dtype=torch.float64, device="cuda"),
                    T=torch.zeros(k * k, dtype=torch.float64, device="cuda"),
                    S=torch.zeros(k * k, dtype=torch.float64, device="cuda"),
                    out=torch.zeros(2, dtype=torch.float64, device="cuda"))
    d, c = bufs(), bufs()
    rd = slra.cross_approx_device(At.data_ptr(), n, n, n, 0, k, k, init.data_ptr(), loops, 1.1, d["I"].data_ptr(),
                                  d["J"].data_ptr(), d["U"].data_ptr(), d["T"].data_ptr(), d["S"].data_ptr())
    slra.cur_residual_factored_device(At.data_ptr(), n, n, n, d["I"].data_ptr(), k, d["J"].data_ptr(), k,
                                      d["T"].data_ptr(), d["S"].data_ptr(), rd, d["out"].data_ptr())
    rc = slra.cross_approx_cauchy_device(x.data_ptr(), y.data_ptr(), n, n, 0, k, k, init.data_ptr(), loops, 1.1,
                                         c["I"].data_ptr(), c["J"].data_ptr(), c["U"].data_ptr(), c["T"].data_ptr(),
                                         c["S"].data_ptr())
    slra.cur_residual_factored_cauchy_device(x.data_ptr(), y.data_ptr(), n, n, c["I"].data_ptr(), k,
                                             c["J"].data_ptr(), k, c["T"].data_ptr(), c["S"].data_ptr(), rc,
                                             c["out"].data_ptr())
    torch.cuda.synchronize()
    assert rd == rc
    for key in ("I", "J", "U", "T", "S", "out"):
        assert torch.equal(d[key], c[key]), key
