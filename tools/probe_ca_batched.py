"""Probe: cost split of the batched C-A kernel (config 5 shape) — one wave of
blocks (one per SM) at 1/2/4 loops: the slope is the per-sweep cost, the
intercept the nucleus + residual factors."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_01391_b200 as slra  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
slra.set_device(0, stream.cuda_stream)
m, k = 256, 32
nb = torch.cuda.get_device_properties(0).multi_processor_count
g = torch.Generator().manual_seed(0)
P = torch.rand(nb, m, 2, dtype=torch.float64, generator=g).cuda()
Q = torch.rand(nb, m, 2, dtype=torch.float64, generator=g).cuda()
Q[..., 0] += 4.0
d = P[:, None, :, :] - Q[:, :, None, :]
A = (0.5 * torch.log((d * d).sum(-1))).contiguous()
init = torch.stack([torch.randperm(m, generator=g)[:k] for _ in range(nb)]).cuda()
I = torch.zeros(nb, k, dtype=torch.int64, device="cuda")
J = torch.zeros(nb, k, dtype=torch.int64, device="cuda")
U = torch.zeros(nb, k * k, dtype=torch.float64, device="cuda")
r = torch.zeros(nb, dtype=torch.int64, device="cuda")
st = torch.zeros(nb, dtype=torch.int32, device="cuda")
rs = torch.zeros(nb, dtype=torch.float64, device="cuda")
ns = torch.zeros(nb, dtype=torch.float64, device="cuda")
for loops in (1, 2, 4):
    def run():
        slra.cross_approx_batched_device(A.data_ptr(), m, m * m, nb, m, m, 0, k, k, init.data_ptr(), loops, 1.1,
                                         I.data_ptr(), J.data_ptr(), U.data_ptr(), r.data_ptr(), st.data_ptr(),
                                         rs.data_ptr(), ns.data_ptr())
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"loops={loops}: {e0.elapsed_time(e1) / 3 * 1e3:.0f} us per wave of {nb} blocks")
