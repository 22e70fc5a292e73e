"""Probe: device time of slra_svd / slra_thin_qr (events on the context's own stream)."""
import ctypes, sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_01391_b200 import capi
lib = capi.load()
stream = torch.cuda.Stream()
ctx = ctypes.c_void_p()
assert lib.slra_ctx_create(0, ctypes.c_void_p(stream.cuda_stream), ctypes.byref(ctx)) == 0

def timeit(fn, reps=3):
    with torch.cuda.stream(stream):
        assert fn() == 0
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            assert fn() == 0
        e1.record(stream)
        stream.synchronize()
    return e0.elapsed_time(e1) / reps

mats = [("rand48", torch.randn(48, 48, dtype=torch.float64)),
        ("graded48", torch.randn(48, 48, dtype=torch.float64) * (0.5 ** torch.arange(48.0, dtype=torch.float64))[None, :]),
        ("rand32", torch.randn(32, 32, dtype=torch.float64)),
        ("rand16", torch.randn(16, 16, dtype=torch.float64))]
if os.path.exists(os.path.join(os.path.dirname(__file__), "R48.npy")):
    mats.append(("config2_R", torch.from_numpy(np.load(os.path.join(os.path.dirname(__file__), "R48.npy")))))
for name, A in mats:
    n = A.shape[0]
    dA = A.t().contiguous().cuda()
    S = torch.empty(n, n, dtype=torch.float64, device="cuda"); T = torch.empty_like(S)
    sig = torch.empty(n, dtype=torch.float64, device="cuda")
    f = lambda: lib.slra_svd(ctx, dA.data_ptr(), n, n, n, S.data_ptr(), n, sig.data_ptr(), T.data_ptr(), n)
    print(name, "svd ms", round(timeit(f), 4))
for m, c in [(4096, 48), (256, 32), (16384, 64), (512, 48), (256, 16)]:
    A = torch.randn(c, m, dtype=torch.float64, device="cuda")
    Q = torch.empty_like(A); R = torch.empty(c, c, dtype=torch.float64, device="cuda")
    f = lambda: lib.slra_thin_qr(ctx, A.data_ptr(), m, m, c, Q.data_ptr(), m, R.data_ptr(), c)
    print("thin_qr", m, c, "ms", round(timeit(f), 4))
