"""Config 5 (batched superfast-multipole LRA) at scale, on the bench's own
inputs: 65,536 blocks in the benchmark, >= 1024 here, generated exactly as
bench.py generates them (per-block reference Rng points and initial rows,
blocks materialised on the device by slra_gen_log_kernel_blocks).

The log-kernel strips are numerically rank deficient (eps-rank ~13 of 32):
their trailing basis vectors are rounding noise in ANY QR implementation,
so the pivots pick among noise directions — chaotically: a 2e-15 relative
perturbation of a strip changes even the oracle's own first pivot in most
trials (check_half_sweeps). The contract there is
(SURVEY.md §7 hard part 1):
  * replay parity: the oracle's adaptive rank, nucleus and residual on the
    GPU's I, J equal the GPU's within 1e-10 ||B||_F plus the conditioning
    term eps ||C|| ||U|| ||R||;
  * quality: the GPU's residual is as small as the oracle's own C-A run;
  * per half-sweep, the selected rows span the strip's well-determined
    subspace as well as the oracle's maxvol does (check_half_sweeps).
On well-posed blocks of the same shape (Gaussian, full-rank strips) the same
kernel must reproduce the oracle's ordered I, J bit for bit in every block.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu
TOL = 1e-10
M, K, LOOPS = 256, 32, 2


@pytest.fixture(scope="module")
def slra():
    import paper_1611_01391_b200 as s
    return s


@pytest.fixture(scope="module")
def bench():
    import bench as b
    return b


def _run_batched(slra, torch, A, init):
    nb = A.shape[0]
    out = dict(I=torch.zeros((nb, K), dtype=torch.int64, device="cuda"),
               J=torch.zeros((nb, K), dtype=torch.int64, device="cuda"),
               U=torch.zeros((nb, K * K), dtype=torch.float64, device="cuda"),
               r=torch.zeros(nb, dtype=torch.int64, device="cuda"),
               st=torch.zeros(nb, dtype=torch.int32, device="cuda"),
               rs=torch.zeros(nb, dtype=torch.float64, device="cuda"),
               ns=torch.zeros(nb, dtype=torch.float64, device="cuda"))
    slra.cross_approx_batched_device(A.data_ptr(), M, M * M, nb, M, M, 0, K, K, init.data_ptr(), LOOPS, 1.1,
                                     out["I"].data_ptr(), out["J"].data_ptr(), out["U"].data_ptr(),
                                     out["r"].data_ptr(), out["st"].data_ptr(), out["rs"].data_ptr(),
                                     out["ns"].data_ptr())
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def _bench_blocks(slra, bench, torch, b0, nb, seed=0):
    px, py, qx, qy, init = bench.config5_host_inputs(slra, seed, b0, nb)
    A = torch.empty(nb, M, M, dtype=torch.float64, device="cuda")
    dev = [torch.from_numpy(a).cuda() for a in (px, py, qx, qy)]
    slra.gen_log_kernel_blocks_device(*[d.data_ptr() for d in dev], nb, M, M, A.data_ptr(), M, M * M)
    torch.cuda.synchronize()
    return A, init, (px, py, qx, qy)


def test_generator_matches_host_recipe(slra, bench, oracle):
    """Device-materialised blocks equal the host testgen recipe to the last ulp of log."""
    import torch
    A, init, (px, py, qx, qy) = _bench_blocks(slra, bench, torch, 5, 4)
    for t in range(4):
        Kb = slra.gen_log_kernel_block(M, M, slra.Rng(slra.Rng.derive_seed(0, 5 + t)))
        dev = A[t].cpu().numpy().T  # column-major block
        assert np.allclose(dev, Kb, rtol=4e-16, atol=0)
        r = slra.Rng(slra.Rng.derive_seed(0, 5 + t))
        for _ in range(4 * M):
            r.uniform()
        assert list(init[t]) == r.distinct_indices(K, M)


def _factored_residual(Kb, I, J, rk):
    """||B - (C T_r S_r^-1)(S_r^T R)||_F with numpy's SVD of G = B(I, J)."""
    G = Kb[np.ix_(I, J)]
    U, s, Vt = np.linalg.svd(G)
    P = Kb[:, J] @ (Vt[:rk].T / s[:rk])
    Q = U[:, :rk].T @ Kb[I, :]
    return np.linalg.norm(Kb - P @ Q)


def test_config5_bench_blocks_parity(slra, bench, oracle):
    """1024 blocks generated as bench.py does: status, adaptive rank, replay
    parity of the fused residual, ||B||, and residual quality vs the oracle's
    own cross_approx on the same blocks."""
    import torch
    nb = 1024
    A, init, _ = _bench_blocks(slra, bench, torch, 0, nb)
    g = _run_batched(slra, torch, A, torch.from_numpy(init).cuda())
    blocks = np.ascontiguousarray(A.cpu().numpy())
    own = bench.oracle_blocks(oracle, blocks, init, os.cpu_count() or 1)
    assert (g["st"] == 0).all() and (own["status"] == 0).all()
    exact = 0
    worst_ratio = 0.0
    for b in range(nb):
        Kb = np.asfortranarray(blocks[b].T)
        Ib, Jb = g["I"][b].tolist(), g["J"][b].tolist()
        assert sorted(set(Ib)) == sorted(Ib) and sorted(set(Jb)) == sorted(Jb)
        exact += (Ib == own["I"][b].tolist() and Jb == own["J"][b].tolist())
        G = Kb[np.ix_(Ib, Jb)]
        rk = oracle.numerical_rank(G, 1e-10, True)
        assert rk == g["r"][b]
        ro = oracle.primitive_cur(Kb, Ib, Jb, rk)
        eo = oracle.cur_evaluate(Kb, Ib, Jb, ro["nucleus"])
        nK = np.linalg.norm(Kb)
        cond = 64 * 2.2e-16 * np.linalg.norm(Kb[:, Jb]) * np.linalg.norm(ro["nucleus"], 2) * np.linalg.norm(Kb[Ib, :])
        eg = np.sqrt(g["rs"][b])
        assert abs(eg - eo) <= TOL * nK + cond, (b, eg, eo)
        assert abs(np.sqrt(g["ns"][b]) - nK) <= 1e-13 * nK
        # the nucleus itself: the oracle's CUR product on the GPU's sets
        Ug = g["U"][b].reshape(K, K).T
        Cg = oracle.cur_reconstruct(Kb, Ib, Jb, Ug)
        Co = oracle.cur_reconstruct(Kb, Ib, Jb, ro["nucleus"])
        assert np.linalg.norm(Cg - Co) <= TOL * nK + cond
        # quality: the GPU's selection approximates the block as well as the
        # oracle's own C-A run does, both evaluated by the same well-conditioned
        # factored evaluator (the oracle's (C U) R carries an eps ||C|| ||U|| ||R||
        # rounding term ~1e-7 ||B|| at r_eff, far above either selection's error)
        en_g = _factored_residual(Kb, Ib, Jb, rk)
        Io, Jo = own["I"][b].tolist(), own["J"][b].tolist()
        en_o = _factored_residual(Kb, Io, Jo, int(own["r"][b]))
        assert abs(eg - en_g) <= TOL * nK, (b, eg, en_g)
        # within the north-star tolerance, or as good as the oracle's own run
        # (the adaptive rank sits at the 1e-10 cut: sigma_11 / sigma_1 ~ 2e-10,
        # so a selection may keep r = 10 where another keeps 11)
        assert en_g <= max(10.0 * en_o, TOL * nK), (b, en_g, en_o)
        worst_ratio = max(worst_ratio, en_g / max(en_o, 1e-300))
        assert eg / nK < 1e-9
    print(f"config-5 bench blocks: {exact}/{nb} with I,J identical to the oracle's own run; "
          f"worst residual ratio gpu/oracle {worst_ratio:.2f}")


def test_config5_well_posed_bit_exact(slra, oracle):
    """Full-rank strips (Gaussian 256 x 256 blocks, k = l = 32, 2 sweeps,
    adaptive r = 32): the same batched kernel reproduces the oracle's ordered
    I and J in every one of 1024 blocks; residuals within 1e-10 ||B||_F."""
    import torch
    nb = 1024
    rng = np.random.default_rng(7)
    blocks = rng.standard_normal((nb, M, M))  # (b, j, i): column-major blocks
    init = np.stack([rng.permutation(M)[:K] for _ in range(nb)]).astype(np.int64)
    g = _run_batched(slra, torch, torch.from_numpy(blocks).cuda(), torch.from_numpy(init).cuda())
    own = oracle.cross_approx_blocks(np.ascontiguousarray(blocks).ctypes.data, nb, M, M, M, M * M, init, K, K, LOOPS,
                                     1.1, os.cpu_count() or 1)
    assert (g["st"] == 0).all() and (own["status"] == 0).all()
    assert np.array_equal(g["I"], own["I"]) and np.array_equal(g["J"], own["J"])
    assert np.array_equal(g["r"], own["r"])
    nK = np.sqrt(g["ns"])
    assert np.all(np.abs(np.sqrt(g["rs"]) - np.sqrt(own["resid_sq"])) <= TOL * nK)


def span_coefficients(strip, sel, tol=1e-10):
    """max_i || u_i pinv(U(sel, :)) ||_2 over the rows u_i of U, the strip's
    leading singular subspace (sigma > tol sigma_1): how much the selected rows
    must be amplified to express every row of the well-determined part of the
    strip. Basis independent (unlike the pivots on the noise directions).
    maxvol's dominance |Q Q(I,:)^-1| <= h bounds it by h sqrt(|I|); the
    oracle's own selections on config-5 / config-3 strips give ~0.7-0.9,
    random row sets 1.6-11."""
    U, sv, _ = np.linalg.svd(strip, full_matrices=False)
    rho = int((sv > tol * sv[0]).sum())
    Ur = U[:, :rho]
    return float(np.linalg.norm(Ur @ np.linalg.pinv(Ur[sel, :]), axis=1).max()), rho


def check_half_sweeps(A, g_trace, o_trace, limit=1.5):
    """Every half-sweep of the GPU's C-A: distinct rows, and a selection that
    spans the strip's well-determined subspace as well as maxvol does
    (span_coefficients <= max(limit, 1.25 x the oracle's own on ITS strip)).
    The pivots themselves are chaotic at the rounding level on these
    rank-deficient strips: perturbing a config-5 strip by 2e-15 relative
    changes even the first pivot of the oracle's own selection in 55 of 60
    trials, so pivot-by-pivot equality is not a meaningful contract there."""
    out = []
    for t, (sg, so) in enumerate(zip(g_trace, o_trace)):
        if t % 2 == 0:  # vertical: J = select_rows_spanning(A(I,:)^T, l)  (cur.cpp:215-224)
            strip, got = A[sg["rows"], :].T, sg["cols"]
            ostrip, oref = A[so["rows"], :].T, so["cols"]
        else:  # horizontal: I = select_rows_spanning(A(:,J), k)  (cur.cpp:227-236)
            strip, got = A[:, sg["cols"]], sg["rows"]
            ostrip, oref = A[:, so["cols"]], so["rows"]
        assert len(set(got)) == len(got)
        cg, rho = span_coefficients(strip, got)
        co, _ = span_coefficients(ostrip, oref)
        assert cg <= max(limit, 1.25 * co), (t, rho, cg, co)
        out.append((rho, round(cg, 3), round(co, 3)))
    return out


@pytest.mark.parametrize("b", range(8))
def test_half_sweep_selection_quality(slra, bench, oracle, b):
    """Per half-sweep of a config-5 block (the CTA-resident C-A kernel, traced)
    against the oracle's own C-A on the same block: see check_half_sweeps."""
    px, py, qx, qy, init = bench.config5_host_inputs(slra, 0, b, 1)
    Kb = np.asfortranarray(bench.config5_host_blocks(px, py, qx, qy)[0].T)
    g = slra.cross_approx(Kb, 0, K, K, list(init[0]), LOOPS, 1.1, slra.Rng(0))
    o = oracle.cross_approx(Kb, 1, K, K, list(init[0]), LOOPS, 1.1, None, oracle.Rng(0))
    print(f"block {b}: (rank, gpu, oracle) span coefficients per half-sweep {check_half_sweeps(Kb, g['trace'], o['trace'])}")


# ---------------------------------------------------------------- edge cases of the batched entries
def _oracle_block(oracle, Kb, init, k, l, loops):
    o = oracle.cross_approx(Kb, 1, k, l, list(init), loops, 1.1, None, oracle.Rng(0))
    G = Kb[np.ix_(o["I"], o["J"])]
    rk = oracle.numerical_rank(G, 1e-10, True)
    return o, rk


def _batched(slra, torch, A, m, n, k, l, init, loops=2):
    nb = A.shape[0]
    out = dict(I=torch.zeros((nb, k), dtype=torch.int64, device="cuda"),
               J=torch.zeros((nb, l), dtype=torch.int64, device="cuda"),
               U=torch.zeros((nb, k * l), dtype=torch.float64, device="cuda"),
               r=torch.zeros(nb, dtype=torch.int64, device="cuda"),
               st=torch.zeros(nb, dtype=torch.int32, device="cuda"),
               rs=torch.zeros(nb, dtype=torch.float64, device="cuda"),
               ns=torch.zeros(nb, dtype=torch.float64, device="cuda"))
    slra.cross_approx_batched_device(A.data_ptr(), m, m * n, nb, m, n, 0, k, l, init.data_ptr(), loops, 1.1,
                                     out["I"].data_ptr(), out["J"].data_ptr(), out["U"].data_ptr(),
                                     out["r"].data_ptr(), out["st"].data_ptr(), out["rs"].data_ptr(),
                                     out["ns"].data_ptr())
    torch.cuda.synchronize()
    return {kk: v.cpu().numpy() for kk, v in out.items()}


@pytest.mark.parametrize("m,n,k,l", [(200, 150, 12, 12), (97, 131, 7, 7), (256, 256, 48, 48), (64, 256, 16, 24)])
def test_batched_ragged_and_wide_shapes(slra, oracle, m, n, k, l):
    """Shapes off the fused path (m, n not multiples of 8; k, l > 32 -> the
    64-column kernel and the separate residual pass; k != l -> the padding
    branch): well-posed Gaussian blocks, I and J bit-exact vs the oracle in
    every block, residuals within 1e-10 ||B||_F."""
    import torch
    rng = np.random.default_rng(m + n + k + l)
    nb = 6
    blocks = rng.standard_normal((nb, n, m))  # (b, j, i): column-major m x n blocks
    init = np.stack([rng.permutation(m)[:k] for _ in range(nb)]).astype(np.int64)
    g = _batched(slra, torch, torch.from_numpy(blocks).cuda(), m, n, k, l, torch.from_numpy(init).cuda())
    for b in range(nb):
        Kb = np.asfortranarray(blocks[b].T)
        o, rk = _oracle_block(oracle, Kb, init[b], k, l, 2)
        assert g["st"][b] == 0
        assert g["I"][b].tolist() == o["I"] and g["J"][b].tolist() == o["J"], b
        assert g["r"][b] == rk
        c = oracle.primitive_cur(Kb, o["I"], o["J"], rk)
        eo = oracle.cur_evaluate(Kb, o["I"], o["J"], c["nucleus"])
        nK = np.linalg.norm(Kb)
        assert abs(np.sqrt(g["rs"][b]) - eo) <= 1e-10 * nK
        assert abs(np.sqrt(g["ns"][b]) - nK) <= 1e-13 * nK


def test_batched_empty_zero_and_failing_blocks(slra, oracle):
    """nblocks = 0 is a no-op; an all-zero block reports its failure per block
    (GeneratorRankFailure, as the reference throws for it) with resid_sq =
    norm_sq = 0 and r = 0; a rank-1 block gets the adaptive rank 1 and an
    exact CUR; neither disturbs the good block beside them."""
    import torch
    m, k = 64, 8
    nb = 3
    rng = np.random.default_rng(3)
    blocks = np.zeros((nb, m, m))
    blocks[1] = rng.standard_normal((m, m))
    u, v = rng.standard_normal(m), rng.standard_normal(m)
    blocks[2] = np.outer(v, u)  # rank 1 (column-major storage of u v^T)
    init = np.stack([rng.permutation(m)[:k] for _ in range(nb)]).astype(np.int64)
    A = torch.from_numpy(blocks).cuda()
    it = torch.from_numpy(init).cuda()
    g0 = _batched(slra, torch, A[:0], m, m, k, k, it[:0])
    assert all(v.size == 0 for v in g0.values())
    g = _batched(slra, torch, A, m, m, k, k, it)
    assert g["st"][0] == 5 and g["st"][1] == 0 and g["st"][2] == 0  # SLRA_ERR_GENERATOR_RANK_FAILURE
    assert g["rs"][0] == g["ns"][0] == 0.0 and g["r"][0] == 0
    with pytest.raises(oracle.GeneratorRankFailure):
        oracle.cross_approx(np.asfortranarray(blocks[0].T), 1, k, k, list(init[0]), 2, 1.1, None, oracle.Rng(0))
    K2 = np.asfortranarray(blocks[2].T)
    assert g["r"][2] == 1 and np.sqrt(g["rs"][2]) <= 1e-13 * np.linalg.norm(K2)
    Kb = np.asfortranarray(blocks[1].T)
    o, rk = _oracle_block(oracle, Kb, init[1], k, k, 2)
    assert g["I"][1].tolist() == o["I"] and g["J"][1].tolist() == o["J"]


def test_batched_host_entry_chunks_and_pageable(slra, bench):
    """The host-streamed entry on a batch that is not a multiple of its chunk,
    from pageable (not page-locked) numpy memory: identical results to the
    device-resident batched call."""
    import torch
    nb = 37
    A, init, _ = _bench_blocks(slra, bench, torch, 100, nb)
    g = _run_batched(slra, torch, A, torch.from_numpy(init).cuda())
    host = np.ascontiguousarray(A.cpu().numpy())
    out = dict(I=np.zeros((nb, K), np.int64), J=np.zeros((nb, K), np.int64), U=np.zeros((nb, K * K)),
               r=np.zeros(nb, np.int64), st=np.zeros(nb, np.int32), rs=np.zeros(nb), ns=np.zeros(nb))
    slra.cross_approx_batched_host(host.ctypes.data, M, M * M, nb, M, M, 0, K, K, init.ctypes.data, LOOPS, 1.1,
                                   *[out[k].ctypes.data for k in ("I", "J", "U", "r", "st", "rs", "ns")])
    for key in ("I", "J", "U", "r", "st", "rs", "ns"):
        assert np.array_equal(out[key], g[key]), key


def _run_logkernel(slra, torch, pts, init, host=False):
    nb = init.shape[0]
    out = dict(I=torch.zeros((nb, K), dtype=torch.int64), J=torch.zeros((nb, K), dtype=torch.int64),
               U=torch.zeros((nb, K * K), dtype=torch.float64), r=torch.zeros(nb, dtype=torch.int64),
               st=torch.zeros(nb, dtype=torch.int32), rs=torch.zeros(nb, dtype=torch.float64),
               ns=torch.zeros(nb, dtype=torch.float64))
    if host:
        hp = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in pts]
        hi = torch.from_numpy(np.ascontiguousarray(init)).pin_memory()
        out = {k: v.pin_memory() for k, v in out.items()}
        slra.cross_approx_batched_logkernel_host(*[a.data_ptr() for a in hp], nb, M, M, 0, K, K, hi.data_ptr(), LOOPS,
                                                 1.1, *[out[k].data_ptr() for k in ("I", "J", "U", "r", "st", "rs",
                                                                                     "ns")])
    else:
        dp = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in pts]
        di = torch.from_numpy(np.ascontiguousarray(init)).cuda()
        out = {k: v.cuda() for k, v in out.items()}
        slra.cross_approx_batched_logkernel_device(*[a.data_ptr() for a in dp], nb, M, M, 0, K, K, di.data_ptr(),
                                                   LOOPS, 1.1, *[out[k].data_ptr() for k in ("I", "J", "U", "r", "st",
                                                                                            "rs", "ns")])
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("host", [False, True])
def test_logkernel_oracle_bit_identical_to_dense(slra, bench, host):
    """The FunctionOracle path (entries evaluated from the points where C-A
    reads them, oracle.hpp:43-54) gives exactly the dense path's results on
    the same bench blocks: the on-the-fly entries are bit-identical to the
    materialised ones, so every selection, nucleus and residual is too. The
    host variant streams the points in eight chunks (uneven last chunk)."""
    import torch
    nb = 1029 if host else 1024
    A, init, pts = _bench_blocks(slra, bench, torch, 4096, nb)
    dense = _run_batched(slra, torch, A, torch.from_numpy(init).cuda())
    lk = _run_logkernel(slra, torch, pts, init, host=host)
    for key in ("I", "J", "U", "r", "st", "rs", "ns"):
        assert np.array_equal(dense[key], lk[key]), key


def test_logkernel_rejects_unsupported_shapes(slra):
    import torch
    z = torch.zeros(64, dtype=torch.float64, device="cuda")
    iz = torch.zeros(64, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        slra.cross_approx_batched_logkernel_device(z.data_ptr(), z.data_ptr(), z.data_ptr(), z.data_ptr(), 1, 12, 12,
                                                   0, 4, 4, iz.data_ptr(), 1, 1.1, *([iz.data_ptr()] * 7))
