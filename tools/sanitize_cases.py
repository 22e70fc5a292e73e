"""Small cases that launch every kernel family of libslra_cuda.so once or a
few times, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck: tools/sanitize.sh). Sizes are chosen so each tool finishes in
minutes; each case checks its result loosely (the parity tests are the
numerical contract). Measurement helper, not product code.
usage: python tools/sanitize_cases.py [case ...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1611_01391_b200 as slra  # noqa: E402

st = torch.cuda.Stream()
torch.cuda.set_stream(st)
slra.set_device(0, st.cuda_stream)


def c1():  # config-1 C-A, primitive_cur (SVD and COD nuclei), residuals
    A = slra.gen_factor_gaussian(256, 256, 8, 1e-8, slra.Rng(3))
    init = slra.Rng(4).distinct_indices(16, 256)
    g = slra.cross_approx(A, 8, 16, 16, init, 3, 1.1, slra.Rng(0))
    e = slra.cur_evaluate(A, g["I"], g["J"], g["nucleus"])
    assert e < 1e-6 * np.linalg.norm(A)
    G = slra.Rng(5).gaussian_matrix(24, 24)
    q = slra.primitive_cur(G, list(range(24)), list(range(24)), 24, qr_nucleus=True)
    assert np.linalg.norm(G @ q["nucleus"] @ G - G) < 1e-9 * np.linalg.norm(G)
    slra.primitive_cur(G, list(range(20)), list(range(24)), 20, qr_nucleus=True)


def c2():  # range finder (sketch plans, CholeskyQR3, Jacobi SVD, tn_skinny, residual stream)
    n = 1024
    rng = slra.Rng(7)
    A = rng.gaussian_matrix(n, 40) @ rng.gaussian_matrix(40, n)
    for H in (slra.take_columns_random(slra.gen_sparse_circulant(n, 4, rng), 48, rng),
              slra.take_columns_random(slra.gen_asph(n, 3, rng), 48, rng)):
        for trunc in (True, False):
            U, V = slra.range_finder(A, H, 32, trunc)
            assert np.all(np.isfinite(U)) and np.all(np.isfinite(V))


def c3():  # tall strips: TSQR, grid maxvol, Cauchy FunctionOracle C-A + residual
    n = 4096
    A = slra.gen_cauchy_block(n, n, slra.Rng(11))
    init = slra.Rng(12).distinct_indices(64, n)
    g = slra.cross_approx(A, 0, 64, 64, init, 2, 1.1, slra.Rng(0))
    e = slra.cur_evaluate(A, g["I"], g["J"], g["nucleus"])
    assert e < 1e-8 * np.linalg.norm(A)


def c4():  # LSR: sketch plans (rows), augmented Gram, cluster Cholesky + refinement, exact path, residuals
    m, d, k = 1 << 14, 96, 1024
    A, b = slra.gen_lsr_gaussian(m, d, 1e-6, slra.Rng(9))
    rp = slra.Rng(10)
    F = slra.make_product([slra.make_sub_identity(rp.distinct_indices(k, m), m), slra.gen_sparse_circulant(m, 2, rp),
                           slra.gen_sign_diagonal(m, rp)])
    rep = slra.sketch_solve(A, b, F, True)
    assert rep["ratio"] < 2.0
    x = slra.solve_exact(A, b)
    assert np.all(np.isfinite(x))
    Ad = np.asfortranarray(A[:4096, :64].copy())
    Ad[:, 63] = Ad[:, 0]  # rank deficient: the ColPivQR min-norm path
    assert np.all(np.isfinite(slra.solve_exact(Ad, b[:4096])))


def c5():  # batched C-A (dense blocks, TMA-staged strips) and the log-kernel FunctionOracle build
    sys.path.insert(0, ROOT)
    import bench
    nb, M, K = 16, 256, 32
    px, py, qx, qy, init = bench.config5_host_inputs(slra, 0, 0, nb)
    dev = [torch.from_numpy(a).cuda() for a in (px, py, qx, qy)]
    A = torch.empty(nb, M, M, dtype=torch.float64, device="cuda")
    slra.gen_log_kernel_blocks_device(*[d.data_ptr() for d in dev], nb, M, M, A.data_ptr(), M, M * M)
    ini = torch.from_numpy(init).cuda()
    outs = [[torch.zeros(s, dtype=t, device="cuda") for s, t in
             (((nb, K), torch.int64), ((nb, K), torch.int64), ((nb, K * K), torch.float64), (nb, torch.int64),
              (nb, torch.int32), (nb, torch.float64), (nb, torch.float64))] for _ in range(2)]
    slra.cross_approx_batched_device(A.data_ptr(), M, M * M, nb, M, M, 0, K, K, ini.data_ptr(), 2, 1.1,
                                     *[o.data_ptr() for o in outs[0]])
    slra.cross_approx_batched_logkernel_device(*[d.data_ptr() for d in dev], nb, M, M, 0, K, K, ini.data_ptr(), 2,
                                               1.1, *[o.data_ptr() for o in outs[1]])
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(outs[0], outs[1]))
    assert int((outs[0][4] != 0).sum()) == 0


def hss():  # HSS leaves / factors / products
    n = 256
    x = np.linspace(0.0, 1.0, n)
    M = np.asfortranarray(1.0 / (1.0 + np.abs(x[:, None] - x[None, :]) * 50.0))
    h = slra.build_hss(M, 3, 8, 1e-6, "svd", slra.Rng(1))
    assert slra.hss_error(h, M, "frobenius") < 1e-3 * np.linalg.norm(M)
    h2 = slra.build_hss(M, 3, 8, 1e-6, "cur_ca", slra.Rng(2))
    assert np.all(np.isfinite(slra.hss_matvec(h2, np.ones(n))))


CASES = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5, "hss": hss}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
        torch.cuda.synchronize()
        print(f"case {nm} ok", flush=True)
