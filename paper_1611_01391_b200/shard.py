"""Multi-GPU drivers for the configs whose hot path shards.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing (NCCL
on the box, gloo in the CPU tests). The reference is single-process; these
drivers compose the single-GPU C-ABI calls around the exchanges §8e names:

* config 3 (C-A on a row-sharded A): per half-sweep one exchange — the k x n
  row strip A(I,:) assembled by an allreduce of per-rank partial gathers
  (every entry has exactly one nonzero contributor, so the sum is exact), or
  the m x l column strip A(:,J) by an allgather of the local slices. The
  selections (TSQR + maxvol) then run replicated on identical inputs, so every
  rank holds the same I, J. Final residual: local partial sums + one allreduce.
* config 4 (sketched LSR on a row-sharded A|b): each rank sketches the rows it
  owns (slra_sketch_rows_shard skips foreign rows), one allreduce of the
  k x (d+1) sketch (bit-exact for the width <= 2 sketches of config 4), a
  replicated solve, and one allreduce of the residual partials.
* config 5 (independent blocks): ``split`` gives each rank a contiguous block
  range; no communication.

Matrices are column-major: an m x n matrix lives in a torch tensor of shape
(n, m) (``t[j, i] = A[i, j]``), so ``data_ptr()`` with ld = m is the layout
the C-ABI takes. ``DeviceOps`` binds the operations to the sm_100a library;
the CPU tests pass an equivalent oracle-backed object to check the
orchestration (ownership, exchanges, ordering) with world_size 2 on gloo.
"""
from __future__ import annotations

from dataclasses import dataclass


def split(total: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous partition: (start, count) of rank's share."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


class Comm:
    """The two collectives the drivers use, over torch.distributed (or none)."""

    def __init__(self, dist=None):
        self.dist = dist if (dist is not None and dist.is_initialized()) else None
        self.world = self.dist.get_world_size() if self.dist else 1
        self.rank = self.dist.get_rank() if self.dist else 0
        # gloo (CPU tests, or several ranks sharing one GPU in the GPU tests)
        # exchanges device tensors through host copies; NCCL takes them as is
        self.host_staged = self.dist is not None and self.dist.get_backend() == "gloo"

    def allreduce_(self, t):
        if self.dist is not None and self.world > 1:
            if self.host_staged and t.is_cuda:
                h = t.cpu()
                self.dist.all_reduce(h)
                t.copy_(h)
            else:
                self.dist.all_reduce(t)
        return t

    def allgather_cols(self, t, counts):
        """Concatenate per-rank (c, m_r) tensors along dim 1 -> (c, sum m_r):
        the column-major m x c strip assembled from row slices."""
        if self.dist is None or self.world == 1:
            return t
        import torch
        dev = t.device
        src = t.cpu() if (self.host_staged and t.is_cuda) else t
        mx = max(counts)
        buf = src.new_zeros((src.shape[0], mx))
        buf[:, : src.shape[1]] = src
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(parts, buf.contiguous())
        return torch.cat([p[:, :c] for p, c in zip(parts, counts)], dim=1).contiguous().to(dev)


class DeviceOps:
    """Operations on CUDA tensors through the C-ABI (paper_1611_01391_b200._slra)."""

    def __init__(self, slra, torch):
        self.s, self.torch = slra, torch
        # the C-ABI kernels and torch.distributed's collectives must share one
        # stream on this rank's device: bind the slra context to torch's
        # current stream (collectives then order after the kernels that write
        # their buffers, with no host synchronisation)
        # (torch's legacy default stream has handle 0, which the C-ABI reads as
        # "make a private stream": pass cudaStreamLegacy = 1 instead)
        handle = torch.cuda.current_stream().cuda_stream or 1
        if slra.stream_ptr() != handle:
            slra.set_device(torch.cuda.current_device(), handle)
        self.stream = handle
        self._check_stream()

    def _check_stream(self):
        assert self.s.stream_ptr() == (self.torch.cuda.current_stream().cuda_stream or 1), \
            "slra context stream != torch current stream: collectives would race the kernels"

    def _f64(self, *shape):
        return self.torch.empty(*shape, dtype=self.torch.float64, device="cuda")

    def ca_blocks(self, seed, b0, nb, m, k, loops, h):
        """Config-5 blocks b0..b0+nb-1: host points / initial rows from the
        reference Rng (per-block seeds), blocks materialised on the device,
        one batched C-A + fused residual launch. Per-block results (device)."""
        import numpy as np
        torch = self.torch
        px, py, qx, qy = (np.empty((nb, m)) for _ in range(4))
        init = np.empty((nb, k), dtype=np.int64)
        self.s.gen_log_kernel_batch(seed, b0, nb, m, m, k, px.ctypes.data, py.ctypes.data, qx.ctypes.data,
                                    qy.ctypes.data, init.ctypes.data)
        dev = [torch.from_numpy(a).cuda() for a in (px, py, qx, qy)]
        A = self._f64(nb, m, m)
        self.s.gen_log_kernel_blocks_device(*[d.data_ptr() for d in dev], nb, m, m, A.data_ptr(), m, m * m)
        init_d = torch.from_numpy(init).cuda()
        out = {"I": torch.empty(nb, k, dtype=torch.int64, device="cuda"),
               "J": torch.empty(nb, k, dtype=torch.int64, device="cuda"),
               "U": self._f64(nb, k * k), "r": torch.empty(nb, dtype=torch.int64, device="cuda"),
               "status": torch.empty(nb, dtype=torch.int32, device="cuda"),
               "resid_sq": self._f64(nb), "norm_sq": self._f64(nb)}
        self.s.cross_approx_batched_device(A.data_ptr(), m, m * m, nb, m, m, 0, k, k, init_d.data_ptr(), loops, h,
                                           out["I"].data_ptr(), out["J"].data_ptr(), out["U"].data_ptr(),
                                           out["r"].data_ptr(), out["status"].data_ptr(), out["resid_sq"].data_ptr(),
                                           out["norm_sq"].data_ptr())
        return out

    def rows_shard(self, W_t, row0, src, coef, width, k, transpose, out=None):
        ncols, mloc = W_t.shape
        if out is None:
            out = self._f64(k, ncols) if transpose else self._f64(ncols, k)
        ldo = ncols if transpose else k
        self.s.sketch_rows_shard_device(W_t.data_ptr(), mloc, row0, mloc, ncols, src.data_ptr(), coef.data_ptr(),
                                        width, k, out.data_ptr(), ldo, transpose)
        return out

    def select(self, S_t, count, h):
        c, m = S_t.shape
        idx = self.torch.empty(count, dtype=self.torch.int64, device="cuda")
        self.s.select_rows_spanning_device(S_t.data_ptr(), m, m, c, count, h, idx.data_ptr(), 0)
        return idx

    def gather_cols(self, A_t, J):
        n, mloc = A_t.shape
        out = self._f64(J.numel(), mloc)
        self.s.gather_cols_device(A_t.data_ptr(), mloc, mloc, n, J.data_ptr(), J.numel(), out.data_ptr(), mloc)
        return out

    def primitive_cur(self, C_t, I, r):
        """Nucleus of G = C(I, :) for the full m x l column strip C."""
        l, m = C_t.shape
        k = I.numel()
        J = self.torch.arange(l, dtype=self.torch.int64, device="cuda")
        U, T, S = self._f64(k, l), self._f64(min(k, l), l), self._f64(min(k, l), k)
        rr = self.s.primitive_cur_device(C_t.data_ptr(), m, m, l, I.data_ptr(), k, J.data_ptr(), l, r,
                                         U.data_ptr(), T.data_ptr(), S.data_ptr())
        return U, T, S, rr

    def cur_residual_partial(self, A_t, C_loc, T, S, R_t, r):
        """(||A_loc - C_loc Tsig Sr^T R||^2, ||A_loc||^2) as a device tensor (2,)."""
        n, mloc = A_t.shape
        l, k = C_loc.shape[0], R_t.shape[1]
        P = self._f64(r, mloc)  # mloc x r
        Q = self._f64(n, r)     # r x n
        self.s.gemm_device(0, 0, mloc, r, l, 1.0, C_loc.data_ptr(), mloc, T.data_ptr(), l, 0.0, P.data_ptr(), mloc)
        self.s.gemm_device(1, 0, r, n, k, 1.0, S.data_ptr(), k, R_t.data_ptr(), k, 0.0, Q.data_ptr(), r)
        out = self.torch.zeros(2, dtype=self.torch.float64, device="cuda")
        self.s.lowrank_residual_device(A_t.data_ptr(), mloc, mloc, n, P.data_ptr(), mloc, Q.data_ptr(), r, r,
                                       out.data_ptr())
        return out

    def lsr_solve(self, FW_t, k, d):
        x = self._f64(d)
        res = self.s.lsr_solve_sketched_device(FW_t.data_ptr(), k, d, x.data_ptr())
        return x, res

    def lsr_residual_partial(self, A_t, b, x):
        d, mloc = A_t.shape
        out = self.torch.zeros(2, dtype=self.torch.float64, device="cuda")
        self.s.lsr_residual_device(A_t.data_ptr(), mloc, mloc, d, b.data_ptr(), x.data_ptr(), out.data_ptr())
        return out


@dataclass
class ShardedCur:
    I: object
    J: object
    nucleus: object
    r: int
    resid_sq: float
    norm_sq: float


def cross_approx(ops, comm, A_t, row0, m, r, k, l, init_rows, loops, h, torch):
    """cross_approx (cur.cpp:201-255) + cur_evaluate(Frobenius) on a row-sharded A.

    A_t: this rank's rows [row0, row0 + m_local) as an (n, m_local) tensor.
    init_rows: the k global initial rows (drawn once on the host exactly as
    cur.cpp:207-209, identical on every rank). Requires k == l (config 3).
    """
    n, mloc = A_t.shape
    if k != l:
        raise ValueError("sharded cross_approx: k == l (no padding branch)")
    counts = [mloc]
    if comm.world > 1:
        counts = [None] * comm.world
        comm.dist.all_gather_object(counts, mloc)
    dev = A_t.device
    I = torch.tensor(list(init_rows), dtype=torch.int64, device=dev)
    ones_k = torch.ones(k, dtype=torch.float64, device=dev)
    J = None
    C_loc = C_full = None
    for _ in range(loops):
        # vertical half-sweep: J = select_rows_spanning(A(I,:)^T, l)
        RT = ops.rows_shard(A_t, row0, I, ones_k, 1, k, transpose=True)  # n x k strip
        comm.allreduce_(RT)
        J = ops.select(RT, l, h)
        # horizontal half-sweep: I = select_rows_spanning(A(:,J), k)
        C_loc = ops.gather_cols(A_t, J)
        C_full = comm.allgather_cols(C_loc, counts)
        I = ops.select(C_full, k, h)
    U, T, S, rr = ops.primitive_cur(C_full, I, r)
    R = ops.rows_shard(A_t, row0, I, ones_k, 1, k, transpose=False)  # k x n strip
    comm.allreduce_(R)
    part = ops.cur_residual_partial(A_t, C_loc, T, S, R, rr)
    comm.allreduce_(part)
    p = part.cpu().tolist()
    return ShardedCur(I, J, U, int(rr), p[0], p[1])


def sketch_solve(ops, comm, A_t, b, row0, d, src, coef, width, k, torch):
    """sketch_solve (lsr.cpp:37-67) on row-sharded (A | b) + the true residual.

    src/coef: the compiled left plan of F (global row indices, LIST order).
    Returns (x_hat, sketched_residual, ||A x_hat - b||).
    """
    dev = A_t.device
    FW = torch.zeros(d + 1, k, dtype=torch.float64, device=dev)  # k x (d+1), column-major
    ops.rows_shard(A_t, row0, src, coef, width, k, transpose=False, out=FW[:d])
    ops.rows_shard(b.reshape(1, -1), row0, src, coef, width, k, transpose=False, out=FW[d:])
    comm.allreduce_(FW)
    x, sres = ops.lsr_solve(FW, k, d)
    part = ops.lsr_residual_partial(A_t, b, x)
    comm.allreduce_(part)
    return x, sres, float(part[0].item()) ** 0.5


def cross_approx_blocks(ops, comm, seed, nblocks, torch, m=256, k=32, loops=2, h=1.1):
    """Config 5 over the ranks: rank r factorises the
    contiguous block range split(nblocks, world, r) of the seeded batch — the
    per-block seeds derive_seed(seed, b) make every block's input and result
    independent of the rank count — with no communication on the data path.
    One allgather of the per-block scalars at the end. Returns a
    (nblocks, 4) float64 tensor: r, ||B - CUR||^2, ||B||^2, status."""
    b0, nb = split(nblocks, comm.world, comm.rank)
    res = ops.ca_blocks(seed, b0, nb, m, k, loops, h)
    loc = torch.stack([res["r"].double(), res["resid_sq"], res["norm_sq"], res["status"].double()], 0)  # (4, nb)
    counts = [split(nblocks, comm.world, r)[1] for r in range(comm.world)]
    return comm.allgather_cols(loc.contiguous(), counts).T.contiguous()
