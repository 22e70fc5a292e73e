"""Measurement of the SURVEY.md §8f rows (beyond BASELINE's five configs):
each row's public entry point on the B200 (host arrays in, host arrays out:
uploads and read-backs inside the timing) against the CPU oracle on the same
inputs and seeds, plus a parity figure. One JSON line per row on stdout.

    python tools/bench_rows.py [--rows hss_svd,hss_ca,...] [--reps 3]

Wall-clock timing of synchronous calls (every entry point blocks on its
result); the oracle is timed once (single-threaded restatement of the
reference algorithm).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle", "build"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import _oracle as o  # noqa: E402
import paper_1611_01391_b200 as s  # noqa: E402
from hss_inputs import cauchy_kernel  # noqa: E402


def timed(fn, reps):
    fn()  # warm-up (arena growth, module load)
    ts = []
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return out, min(ts)


def once(fn):
    t0 = time.perf_counter()
    out = fn()
    return out, time.perf_counter() - t0


def hss_parity(h, ho, M):
    ranks = [b["F"].shape[1] for b in h["off"]] == [b["F"].shape[1] for b in ho["off"]]
    err = max(np.linalg.norm(b["F"] @ b["H"] - bo["F"] @ bo["H"]) for b, bo in zip(h["off"], ho["off"]))
    return {"ranks_equal": ranks, "max_block_diff_rel": err / np.linalg.norm(M)}


def row_hss_svd(reps):
    n, L, r, tol = 1024, 3, 24, 1e-10
    M = cauchy_kernel(n)
    h, tg = timed(lambda: s.build_hss(M, L, r, tol, "svd", s.Rng(0)), reps)
    ho, tc = once(lambda: o.build_hss(M, L, r, tol, "svd", o.Rng(0)))
    return {"row": "build_hss(Svd)", "config": f"cauchy n={n} L={L} r={r} tol={tol}", "gpu_s": tg, "cpu_s": tc,
            **hss_parity(h, ho, M)}


def row_hss_ca(reps):
    n, L, r, tol = 4096, 5, 16, 1e-8
    M = cauchy_kernel(n)
    h, tg = timed(lambda: s.build_hss(M, L, r, tol, "cur_ca", s.Rng(50)), reps)
    ho, tc = once(lambda: o.build_hss(M, L, r, tol, "cur_ca", o.Rng(50)))
    # at ranks near the blocks' numerical rank the C-A strips are rank
    # deficient and the selections ill-posed (any two QR implementations
    # diverge there), so the comparison is the achieved accuracy
    nM = np.linalg.norm(M)
    return {"row": "build_hss(CurCa)", "config": f"cauchy n={n} L={L} r={r} tol={tol}", "gpu_s": tg, "cpu_s": tc,
            "reads_fraction": h["accesses"] / n / n, "hss_err_rel": s.hss_error(h, M, "frobenius") / nM,
            "oracle_hss_err_rel": o.hss_error(ho, M, "frobenius") / nM, **hss_parity(h, ho, M)}


def row_hss_matvec(reps):
    import torch
    n, L, r, tol = 8192, 6, 16, 1e-8
    M = cauchy_kernel(n)
    ho = o.build_hss(M, L, r, tol, "cur_ca", o.Rng(1))
    x = np.random.default_rng(0).standard_normal(n)
    _, tc = once(lambda: o.hss_matvec(ho, x))
    dx = torch.tensor(x, device="cuda")
    dy = torch.empty_like(dx)
    t_mv = s.hss_matvec_timed(M, L, r, tol, "cur_ca", s.Rng(1), dx.data_ptr(), dy.data_ptr(), 500)
    y = dy.cpu().numpy()
    R = o.hss_reconstruct(ho)
    return {"row": "hss_matvec (device-resident)", "config": f"cauchy n={n} L={L} r={r}", "gpu_s": t_mv,
            "cpu_s": tc, "dense_gemv_bytes": 8 * n * n,
            "rel_diff_vs_oracle_matvec": float(np.linalg.norm(y - o.hss_matvec(ho, x)) / np.linalg.norm(R @ x))}


def row_premult(reps):
    m = n = 4096
    M = o.gen_factor_gaussian(m, n, 32, 1e-8, o.Rng(3))
    rp, ro = s.Rng(9), o.Rng(9)
    Hp = s.take_columns_random(s.gen_sparse_circulant(n, 4, rp), 48, rp)
    Ho = o.take_columns_random(o.gen_sparse_circulant(n, 4, ro), 48, ro)
    sp, so = rp.distinct_indices(256, m), ro.distinct_indices(256, m)
    Fp = s.make_product([s.make_sub_identity(sp, m), s.gen_sparse_circulant(m, 2, rp), s.gen_sign_diagonal(m, rp)])
    Fo = o.make_product([o.make_sub_identity(so, m), o.gen_sparse_circulant(m, 2, ro), o.gen_sign_diagonal(m, ro)])
    (U, V), tg = timed(lambda: s.lra_premult(M, Fp, Hp, 32, True), reps)
    (Uo, Vo), tc = once(lambda: o.lra_premult(M, Fo, Ho, 32, True))
    return {"row": "lra_premult(TruncatedRankR)", "config": "4096^2 rank-32+1e-8, H: Z_f s=4 l=48, F: 256 rows s=2",
            "gpu_s": tg, "cpu_s": tc,
            "product_diff_rel": float(np.linalg.norm(U @ V - Uo @ Vo) / np.linalg.norm(M))}


def row_two_stage(reps):
    rng = o.Rng(11)
    U, V = rng.gaussian_matrix(4096, 48), rng.gaussian_matrix(48, 4096)
    (Ug, Vg), tg = timed(lambda: s.two_stage_truncate(U, V, 32), reps)
    (Uo, Vo), tc = once(lambda: o.two_stage_truncate(U, V, 32))
    return {"row": "two_stage_truncate", "config": "U 4096x48, V 48x4096 -> r=32", "gpu_s": tg, "cpu_s": tc,
            "product_diff_rel": float(np.linalg.norm(Ug @ Vg - Uo @ Vo) / np.linalg.norm(U @ V))}


def row_retries(reps):
    m, d, k = 1 << 18, 128, 2048
    A, b = o.gen_lsr_gaussian(m, d, 1e-6, o.Rng(7))

    def mk(lib, seed):
        r = lib.Rng(seed)
        sel = r.distinct_indices(k, m)
        F = lib.make_product([lib.make_sub_identity(sel, m), lib.gen_sparse_circulant(m, 2, r),
                              lib.gen_sign_diagonal(m, r)])
        return F, r

    def gpu():
        F, r = mk(s, 5)
        return s.solve_with_retries(A, b, F, [], 2, 2.0, r)

    def cpu():
        F, r = mk(o, 5)
        return o.solve_with_retries(A, b, F, [], 2, 2.0, r)

    rp, tg = timed(gpu, reps)
    ro, tc = once(cpu)
    return {"row": "solve_with_retries", "config": f"m=2^18 d={d} k={k} circulant s=2", "gpu_s": tg, "cpu_s": tc,
            "attempts": rp["attempts"], "validated": rp["validated"], "attempts_equal": rp["attempts"] == ro["attempts"],
            "x_diff_rel": float(np.linalg.norm(rp["x_hat"] - ro["x_hat"]) / np.linalg.norm(ro["x_hat"]))}


def row_leverage(reps):
    n, r, k = 2048, 16, 96
    M = o.gen_factor_gaussian(n, n, r, 1e-8, o.Rng(13))
    c, tg = timed(lambda: s.cur_via_leverage(M, r, k, k, 1.0, 1.0, "exactly", s.uniform_scores(n), s.Rng(3)), reps)
    co, tc = once(lambda: o.cur_via_leverage(M, r, k, k, 1.0, 1.0, "exactly", o.uniform_scores(n), o.Rng(3)))
    Cp = M[:, c["J"]] @ c["nucleus"] @ M[c["I"], :]
    Co = M[:, co["J"]] @ co["nucleus"] @ M[co["I"], :]
    return {"row": "cur_via_leverage (uniform scores)", "config": f"{n}^2 rank-{r}+1e-8 k=l={k}", "gpu_s": tg,
            "cpu_s": tc, "sets_equal": c["I"] == co["I"] and c["J"] == co["J"],
            "product_diff_rel": float(np.linalg.norm(Cp - Co) / np.linalg.norm(M))}


def row_large_svd(reps):
    A = o.Rng(17).gaussian_matrix(1024, 512)
    (S, sig, T), tg = timed(lambda: s.svd(A), reps)
    (So, sigo, To), tc = once(lambda: o.svd(A))
    return {"row": "svd (multi-CTA Jacobi)", "config": "1024 x 512 Gaussian", "gpu_s": tg, "cpu_s": tc,
            "sigma_rel_diff": float(np.max(np.abs(sig - sigo)) / sigo[0])}


def row_leverage_full(reps):
    n, r, k = 768, 12, 64
    M = o.gen_factor_gaussian(n, n, r, 1e-8, o.Rng(14))
    c, tg = timed(lambda: s.cur_via_leverage(M, r, k, k, 1.0, 1.0, "exactly", None, s.Rng(4)), reps)
    co, tc = once(lambda: o.cur_via_leverage(M, r, k, k, 1.0, 1.0, "exactly", None, o.Rng(4)))
    Cp = M[:, c["J"]] @ c["nucleus"] @ M[c["I"], :]
    Co = M[:, co["J"]] @ co["nucleus"] @ M[co["I"], :]
    return {"row": "cur_via_leverage (dense-SVD scores)", "config": f"{n}^2 rank-{r}+1e-8 k=l={k}", "gpu_s": tg,
            "cpu_s": tc, "sets_equal": c["I"] == co["I"] and c["J"] == co["J"],
            "product_diff_rel": float(np.linalg.norm(Cp - Co) / np.linalg.norm(M))}


ROWS = {"hss_svd": row_hss_svd, "hss_ca": row_hss_ca, "hss_matvec": row_hss_matvec, "premult": row_premult,
        "two_stage": row_two_stage, "retries": row_retries, "leverage": row_leverage, "leverage_full": row_leverage_full, "svd_large": row_large_svd}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default=",".join(ROWS))
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for name in a.rows.split(","):
        try:
            rec = ROWS[name](a.reps)
            rec["speedup"] = rec["cpu_s"] / rec["gpu_s"]
        except Exception as e:  # report and continue with the next row
            rec = {"row": name, "error": f"{type(e).__name__}: {e}"}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
