"""The multi-GPU drivers (shard.py) on the device: two gloo ranks sharing one
B200 (host-staged collectives, so no kernel waits on another rank), each
running its shard through shard.DeviceOps -> the sm_100a C-ABI. Results must
equal the single-GPU path on the full matrix and the oracle:
* config-3 shape: identical I, J (the all-reduced / all-gathered strips are
  bit-identical to the single-GPU strips, and the selections are the same
  kernels), residual within 1e-12 ||A||_F;
* config-4 shape: the sharded sketch-and-solve equals slra_sketch_solve.
"""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(rank, world, port, name, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1611_01391_b200 as slra
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        slra.set_device(0, stream.cuda_stream)
        q.put((rank, WORKERS[name](slra, torch, dist, rank, world)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, traceback.format_exc() + repr(e)))
    finally:
        dist.destroy_process_group()


def _spawn(name, world=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(120)
    return out


N3, K3 = 4096, 64


def _cauchy_points(slra, n, seed):
    r = slra.Rng(seed)
    x = [r.uniform() for _ in range(n)]
    y = [2.0 + r.uniform() for _ in range(n)]
    return x, y


def _ca_worker(slra, torch, dist, rank, world):
    from paper_1611_01391_b200 import shard
    x, y = _cauchy_points(slra, N3, 5)
    row0, mloc = shard.split(N3, world, rank)
    xd = torch.tensor(x[row0:row0 + mloc], dtype=torch.float64, device="cuda")
    yd = torch.tensor(y, dtype=torch.float64, device="cuda")
    At = (1.0 / (xd[None, :] - yd[:, None])).contiguous()
    init = slra.Rng(77).distinct_indices(K3, N3)
    res = shard.cross_approx(shard.DeviceOps(slra, torch), shard.Comm(dist), At, row0, N3, 0, K3, K3, init, 5, 1.1,
                             torch)
    return {"I": res.I.tolist(), "J": res.J.tolist(), "r": res.r, "rs": res.resid_sq, "ns": res.norm_sq}


M4, D4, K4 = 1 << 16, 64, 1024


def _lsr_data(torch, row0, mloc):
    g = torch.Generator(device="cpu").manual_seed(3)
    A = torch.randn(M4, D4, dtype=torch.float64, generator=g)
    x0 = torch.randn(D4, dtype=torch.float64, generator=g)
    b = A @ x0 + 1e-6 * torch.randn(M4, dtype=torch.float64, generator=g)
    return (A[row0:row0 + mloc].T.contiguous().cuda(), b[row0:row0 + mloc].contiguous().cuda())


def _lsr_plan(slra):
    rs = slra.Rng(8)
    F = slra.make_product([slra.make_sub_identity(rs.distinct_indices(K4, M4), M4),
                           slra.gen_sparse_circulant(M4, 2, rs), slra.gen_sign_diagonal(M4, rs)])
    return F.plan("left")


def _lsr_worker(slra, torch, dist, rank, world):
    from paper_1611_01391_b200 import shard
    row0, mloc = shard.split(M4, world, rank)
    At, b = _lsr_data(torch, row0, mloc)
    p = _lsr_plan(slra)
    src = torch.tensor(p["src"], dtype=torch.int64, device="cuda")
    coef = torch.tensor(p["coef"], dtype=torch.float64, device="cuda")
    x, sres, tres = shard.sketch_solve(shard.DeviceOps(slra, torch), shard.Comm(dist), At, b, row0, D4, src, coef,
                                       p["width"], K4, torch)
    return {"x": x.tolist(), "sres": sres, "tres": tres}


NB5 = 301  # config-5 blocks for the split test (ragged over two ranks)


def _blocks_worker(slra, torch, dist, rank, world):
    from paper_1611_01391_b200 import shard
    out = shard.cross_approx_blocks(shard.DeviceOps(slra, torch), shard.Comm(dist), 0, NB5, torch)
    return out.cpu().numpy().tolist()


WORKERS = {"ca": _ca_worker, "lsr": _lsr_worker, "blocks": _blocks_worker}


@pytest.fixture(scope="module")
def slra():
    import paper_1611_01391_b200 as s
    return s


def test_sharded_cross_approx_two_ranks_one_gpu(slra, oracle):
    out = _spawn("ca")
    assert all(isinstance(v, dict) for v in out.values()), out
    a, b = out[0], out[1]
    assert a["I"] == b["I"] and a["J"] == b["J"]
    # single-GPU path on the full matrix
    x, y = _cauchy_points(slra, N3, 5)
    A = 1.0 / (np.array(x)[:, None] - np.array(y)[None, :])
    init = slra.Rng(77).distinct_indices(K3, N3)
    g = slra.cross_approx(A, 0, K3, K3, init, 5, 1.1, slra.Rng(0))
    assert a["I"] == g["I"] and a["J"] == g["J"] and a["r"] == g["r"]
    nA = np.linalg.norm(A)
    # same factored evaluation (C Tsig)(Sr^T R) on the full matrix; the
    # unfactored (C U) R carries an eps * ||C|| ||U|| ||R|| ~ 1e-6 ||A||
    # rounding term at this conditioning (sigma_r ~ 1e-10 sigma_1)
    p = slra.primitive_cur(A, g["I"], g["J"], 0)
    ef = slra.cur_evaluate_factored(A, g["I"], g["J"], p["tsig"], p["sr"])
    assert abs(np.sqrt(a["rs"]) - ef) <= 1e-12 * nA
    assert abs(np.sqrt(a["ns"]) - nA) <= 1e-13 * nA
    # replay parity against the oracle on the same I, J
    rk = oracle.numerical_rank(A[np.ix_(a["I"], a["J"])], 1e-10, True)
    assert rk == a["r"]


def test_sharded_sketch_solve_two_ranks_one_gpu(slra):
    import torch
    out = _spawn("lsr")
    assert all(isinstance(v, dict) for v in out.values()), out
    At, b = _lsr_data(torch, 0, M4)
    p = _lsr_plan(slra)
    dev = dict(src=torch.tensor(p["src"], dtype=torch.int64, device="cuda"),
               coef=torch.tensor(p["coef"], dtype=torch.float64, device="cuda"),
               q=torch.tensor(p["q"], dtype=torch.int32, device="cuda"))
    x = torch.zeros(D4, dtype=torch.float64, device="cuda")
    sres = slra.sketch_solve_device(At.data_ptr(), M4, M4, D4, b.data_ptr(), dev["src"].data_ptr(),
                                    dev["coef"].data_ptr(), dev["q"].data_ptr(), p["width"], p["tree"], K4,
                                    x.data_ptr())
    xs = np.array(out[0]["x"])
    # the all-reduced sketch is bit-identical (width 2), so the solve is too
    assert np.array_equal(xs, x.cpu().numpy())
    assert out[0]["sres"] == sres
    r = (At.T @ x - b).norm().item()
    assert abs(out[0]["tres"] - r) <= 1e-10 * b.norm().item()


def test_config5_block_split_two_ranks_one_gpu(slra):
    """Config 5 split over two ranks sharing the GPU: the gathered per-block
    ranks, residuals and norms equal the single-process batched run bit for bit."""
    import torch
    from paper_1611_01391_b200 import shard
    out = _spawn("blocks")
    assert all(isinstance(v, list) for v in out.values()), out
    single = shard.cross_approx_blocks(shard.DeviceOps(slra, torch), shard.Comm(None), 0, NB5, torch).cpu().numpy()
    for r in (0, 1):
        assert np.array_equal(np.array(out[r]), single)
    assert (single[:, 3] == 0).all()


def test_comm_single_rank_sketch_solve(slra):
    """The C-ABI's NCCL communicator (slra_comm_*), one rank on this GPU: the
    sharded driver sketch_solve_sharded (one allreduce of the sketch, one of
    the residual partials) equals sketch_solve on the same data."""
    import torch
    if not slra.comm_available():
        pytest.skip("libnccl.so.2 not loadable")
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    slra.set_device(0, stream.cuda_stream)
    comm = slra.comm_init(1, 0, slra.comm_unique_id())
    try:
        m, d, k = 20000, 48, 1024
        rng = slra.Rng(31)
        A, b = slra.gen_lsr_gaussian(m, d, 1e-6, rng)
        F = slra.make_product([slra.make_sub_identity(rng.distinct_indices(k, m), m),
                               slra.gen_sparse_circulant(m, 2, rng), slra.gen_sign_diagonal(m, rng)])
        At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
        bd = torch.from_numpy(b).cuda()
        got = slra.sketch_solve_sharded(comm, At.data_ptr(), m, m, d, bd.data_ptr(), 0, m, F, True)
        ref = slra.sketch_solve(A, b, F, True)
        assert np.array_equal(got["x_hat"], ref["x_hat"])
        assert abs(got["true_residual"] - ref["true_residual"]) <= 1e-12 * np.linalg.norm(b)
        # allreduce / allgather on one rank are copies
        x = torch.arange(10, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        slra.comm_allreduce_sum(comm, x.data_ptr(), y.data_ptr(), 10)
        slra.comm_allgather(comm, x.data_ptr(), y.data_ptr(), 10)
        torch.cuda.synchronize()
        assert torch.equal(x, y)
    finally:
        slra.comm_destroy(comm)
