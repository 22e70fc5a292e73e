"""CPU-side checks of the product (no GPU needed):

* the C-ABI library loads and exports every symbol include/slra_cuda.h declares;
* without a device every entry point fails loudly (no CPU fallback);
* the host layer's Rng / generators are bit-identical to the oracle's;
* the sketch-plan compiler (host C++) reproduces the reference operators
  exactly: evaluating a compiled plan in the reference's order equals the
  oracle's full-operator application bit for bit.
"""
import ctypes
import math
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def slra():
    import paper_1611_01391_b200 as s
    return s


def test_library_exports_every_declared_symbol():
    from paper_1611_01391_b200 import capi
    protos = capi.declared_functions()
    assert len(protos) >= 25
    lib = capi.load()  # raises AttributeError on a missing symbol
    for name, _, _ in protos:
        assert hasattr(lib, name)
    assert lib.slra_status_string(capi.STATUS["SLRA_ERR_GENERATOR_RANK_FAILURE"]).startswith(b"primitive_cur")


def test_status_codes_match_header():
    from paper_1611_01391_b200 import capi
    text = open(capi.HEADER).read()
    for k, v in capi.STATUS.items():
        assert f"{k} = {v}" in text


def test_host_library_links_cabi():
    lib = os.path.join(ROOT, "paper_1611_01391_b200", "lib", "libslra.so")
    assert os.path.exists(lib)
    out = os.popen(f"ldd {lib}").read()
    assert "libslra_cuda.so" in out


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_no_cpu_fallback(slra):
    from paper_1611_01391_b200 import capi
    lib = capi.load()
    ctx = ctypes.c_void_p()
    assert lib.slra_ctx_create(0, None, ctypes.byref(ctx)) == capi.STATUS["SLRA_ERR_NO_DEVICE"]
    with pytest.raises(slra.DeviceError):
        slra.thin_qr(np.eye(3))
    with pytest.raises(slra.DeviceError):
        slra.cross_approx(np.eye(8), 1, 2, 2, [0, 1], 1, 1.1, slra.Rng(0))
    # the §8f rows fail the same way (no host path behind them)
    rng = slra.Rng(1)
    with pytest.raises(slra.DeviceError):
        slra.build_hss(np.eye(16), 2, 2, 1e-6, "svd", rng)
    with pytest.raises(slra.DeviceError):
        slra.lra_premult(np.eye(8), slra.gen_gaussian(4, 8, rng), slra.gen_gaussian(8, 3, rng), 2)
    with pytest.raises(slra.DeviceError):
        slra.cur_via_leverage(np.eye(8), 1, 2, 2, 1.0, 1.0, "exactly", slra.uniform_scores(8), rng)
    with pytest.raises(slra.DeviceError):
        slra.gen_inverse_bidiagonal(8, rng).apply(np.eye(8))


def test_shared_libstdcxx_and_import_order(oracle):
    """libslra.so and the binding link the shared libstdc++ (a static copy
    crashes iostream/locale use once another C++ extension is loaded)."""
    for lib in (os.path.join(ROOT, "paper_1611_01391_b200", "lib", "libslra.so"),):
        assert "libstdc++.so.6" in os.popen(f"readelf -d {lib}").read()
    import paper_1611_01391_b200 as s  # imported after the oracle (conftest loads it first)
    h = s.hss_deserialize("hss 4 1 2 0 0 1 0 leaf 0 0 2 2 1 2 3 4")
    assert h["n"] == 4 and h["diag"][0][2].tolist() == [[1.0, 3.0], [2.0, 4.0]]
    assert s.hss_deserialize(s.hss_serialize(h))["diag"][0][2].tolist() == [[1.0, 3.0], [2.0, 4.0]]


def test_rng_bit_identical(slra, oracle):
    for seed in (0, 1, 12345, 2**63 + 7):
        a, b = slra.Rng(seed), oracle.Rng(seed)
        assert [a.next_u64() for _ in range(50)] == [b.next_u64() for _ in range(50)]
        assert [a.gaussian() for _ in range(50)] == [b.gaussian() for _ in range(50)]
        assert a.permutation(97) == b.permutation(97)
        assert a.distinct_indices(40, 1000) == b.distinct_indices(40, 1000)
        assert np.array_equal(a.gaussian_matrix(7, 5), b.gaussian_matrix(7, 5))
        assert a.uniform_index(13) == b.uniform_index(13)
    for master, stream in [(0, 0), (5, 17), (2**64 - 1, 3)]:
        assert slra.Rng.derive_seed(master, stream) == oracle.Rng.derive_seed(master, stream)


def test_generators_bit_identical(slra, oracle):
    assert np.array_equal(slra.gen_factor_gaussian(256, 256, 8, 1e-8, slra.Rng(3)),
                          oracle.gen_factor_gaussian(256, 256, 8, 1e-8, oracle.Rng(3)))
    Ap, bp = slra.gen_lsr_gaussian(500, 12, 1e-6, slra.Rng(4))
    Ao, bo = oracle.gen_lsr_gaussian(500, 12, 1e-6, oracle.Rng(4))
    assert np.array_equal(Ap, Ao) and np.array_equal(bp, bo)
    # config 3 recipe: x ~ U[0,1] then y ~ U[2,3]
    r = oracle.Rng(5)
    x = np.array([r.uniform() for _ in range(300)])
    y = np.array([2.0 + r.uniform() for _ in range(200)])
    assert np.array_equal(slra.gen_cauchy_block(300, 200, slra.Rng(5)), 1.0 / (x[:, None] - y[None, :]))


def _eval_plan(plan, X):
    """Evaluate a compiled plan over the rows of X in the kernel's order."""
    w, cnt, tree = plan["width"], plan["count"], plan["tree"]
    src = np.array(plan["src"], dtype=np.int64).reshape(cnt, w)
    coef = np.array(plan["coef"]).reshape(cnt, w)
    out = np.zeros((cnt, X.shape[1]))
    for t in range(cnt):
        z = [coef[t, s] * X[src[t, s]] for s in range(w)]
        if tree == 0:
            acc = z[0]
            for s in range(1, w):
                acc = acc + z[s]
            out[t] = acc
        else:
            y = list(z)
            ln = w
            while ln > 1:
                h = ln // 2
                for base in range(0, w, ln):
                    for i in range(h):
                        a, b = y[base + i], y[base + i + h]
                        y[base + i], y[base + i + h] = a + b, a - b
                ln = h
            out[t] = y[plan["q"][t]]
    return out


@pytest.mark.parametrize("n", [8, 64, 256])
def test_plan_compiler_matches_reference_operators(slra, oracle, n):
    seed = 900 + n
    rp, ro = slra.Rng(seed), oracle.Rng(seed)
    pairs = [
        (slra.gen_permutation(n, rp), oracle.gen_permutation(n, ro)),
        (slra.gen_sign_diagonal(n, rp), oracle.gen_sign_diagonal(n, ro)),
        (slra.make_abridged_hadamard(n, 3), oracle.make_abridged_hadamard(n, 3)),
        (slra.gen_sparse_circulant(n, 4, rp), oracle.gen_sparse_circulant(n, 4, ro)),
        (slra.gen_asph(n, 3, rp), oracle.gen_asph(n, 3, ro)),
        (slra.gen_aph(n, 2, rp), oracle.gen_aph(n, 2, ro)),
    ]
    l = max(1, n // 8)
    pairs.append((slra.take_columns_random(slra.gen_asph(n, 3, rp), l, rp),
                  oracle.take_columns_random(oracle.gen_asph(n, 3, ro), l, ro)))
    pairs.append((slra.take_columns_random(slra.gen_sparse_circulant(n, 4, rp), l, rp),
                  oracle.take_columns_random(oracle.gen_sparse_circulant(n, 4, ro), l, ro)))
    sel_p, sel_o = rp.distinct_indices(l, n), ro.distinct_indices(l, n)
    pairs.append((slra.make_product([slra.make_sub_identity(sel_p, n), slra.gen_sparse_circulant(n, 2, rp),
                                     slra.gen_sign_diagonal(n, rp)]),
                  oracle.make_product([oracle.make_sub_identity(sel_o, n), oracle.gen_sparse_circulant(n, 2, ro),
                                       oracle.gen_sign_diagonal(n, ro)])))
    M = oracle.Rng(seed + 1).gaussian_matrix(5, n)  # right side: columns of M
    for p, o in pairs:
        W = oracle.Rng(seed + 2).gaussian_matrix(p.cols(), 3)
        if p.kind() != "column_slice":  # ColumnSlice is applied from the right only
            assert np.array_equal(_eval_plan(p.plan("left"), W), o.apply(W)), p.kind()
        if p.rows() == n:
            right = _eval_plan(p.plan("right"), M.T).T
            assert np.array_equal(right, oracle.apply(o, M, "right")), p.kind()


def test_plan_rejects_two_combining_factors(slra):
    op = slra.make_product([slra.make_abridged_hadamard(16, 2), slra.make_abridged_hadamard(16, 2)])
    with pytest.raises(ValueError):
        op.plan("left")


# ---------------------------------------------------------------- INTEGRATION.md glue
def build_integration_example(tmp_path):
    """Compile the reference-side glue of INTEGRATION.md §2-3 (b200.hpp + the
    SLRA_B200 cross_approx definition, tests/integration/) against the C-ABI
    header, linking libslra_cuda.so only — what a maintainer's build adds."""
    import subprocess
    src = os.path.join(ROOT, "tests", "integration")
    lib = os.path.join(ROOT, "paper_1611_01391_b200", "lib")
    exe = str(tmp_path / "ca_dispatch")
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", src,
                    os.path.join(src, "cur_dispatch.cpp"), os.path.join(src, "main.cpp"), "-o", exe, "-L", lib,
                    "-lslra_cuda", f"-Wl,-rpath,{lib}"], check=True)
    return exe


def write_integration_input(path, A, init, loops, r):
    import numpy as np
    m, n = A.shape
    with open(path, "wb") as f:
        np.array([m, n, len(init), loops, r], dtype=np.int64).tofile(f)
        np.asfortranarray(A).T.astype(np.float64).tofile(f)  # column-major
        np.array(init, dtype=np.int64).tofile(f)


def test_integration_glue_compiles_and_fails_loudly_without_gpu(tmp_path):
    import subprocess
    import numpy as np
    exe = build_integration_example(tmp_path)
    A = np.random.default_rng(0).standard_normal((64, 48))
    inp = str(tmp_path / "in.bin")
    write_integration_input(inp, A, list(range(8)), 2, 4)
    p = subprocess.run([exe, inp], capture_output=True, text=True)
    import torch
    if torch.cuda.is_available():
        assert p.returncode == 0, p.stdout + p.stderr
    else:
        # no CPU fallback: the C-ABI refuses, the glue raises
        assert p.returncode == 3 and "no sm_100 device" in p.stdout, p.stdout + p.stderr
