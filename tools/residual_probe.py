"""Device time of the streaming residual ||A - P Q||_F (residual_stream_kernel)
at the config-2 shape (4096^2, inner 32) and the config-3 shape (16384^2,
inner 6), CUDA events over many launches with inputs larger than L2
(rotating A buffers). usage: [LD_LIBRARY_PATH=variant/lib] python tools/residual_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_01391_b200 as slra  # noqa: E402

st = torch.cuda.Stream()
torch.cuda.set_stream(st)
slra.set_device(0, st.cuda_stream)
for (m, n, r, nbuf) in [(4096, 4096, 32, 4), (16384, 16384, 6, 1)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    As = [torch.randn(n, m, device="cuda", dtype=torch.float64, generator=g) for _ in range(nbuf)]  # col-major m x n
    P = torch.randn(r, m, device="cuda", dtype=torch.float64, generator=g)
    Q = torch.randn(n, r, device="cuda", dtype=torch.float64, generator=g)
    out = torch.zeros(2, device="cuda", dtype=torch.float64)

    def run(A):
        slra.lowrank_residual_device(A.data_ptr(), m, m, n, P.data_ptr(), m, Q.data_ptr(), r, r, out.data_ptr())
    for A in As:
        run(A)
    torch.cuda.synchronize()
    reps = 40 if m == 4096 else 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        run(As[i % nbuf])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    fl = 2.0 * m * n * r
    print(f"{m}x{n} inner {r}: {us:.1f} us/launch (incl. reduce), {fl / us / 1e6:.2f} TFLOP/s "
          f"({fl / us / 1e6 / 37.21:.1%} of 37.21), {8.0 * m * n / us / 1e3:.0f} GB/s of A")
