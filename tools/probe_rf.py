"""Probe: per-kernel device time of one config-2 range finder; SVD of the actual sketch R."""
import ctypes, sys, os
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_1611_01391_b200 as slra
from paper_1611_01391_b200 import capi
slra.set_device(0, torch.cuda.current_stream().cuda_stream)
w = bench.Config2(slra, torch, 0)
w.step(); torch.cuda.synchronize()
slra.set_timing(True)
w.step(); torch.cuda.synchronize()
print("one step:", slra.timing_report())
slra.set_timing(False)
# SVD of the real R
lib = capi.load()
ctx = ctypes.c_void_p()
assert lib.slra_ctx_create(0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(ctx)) == 0
name, p, d = w.plans[1]
n, l = 4096, 48
MH = torch.empty(l, n, dtype=torch.float64, device="cuda")
st = lib.slra_sketch_cols(ctx, w.At.data_ptr(), n, n, n, d["src"].data_ptr(), d["coef"].data_ptr(), d["q"].data_ptr(), p["width"], p["tree"], l, MH.data_ptr(), n)
Q = torch.empty_like(MH); R = torch.empty(l, l, dtype=torch.float64, device="cuda")
st2 = lib.slra_thin_qr(ctx, MH.data_ptr(), n, n, l, Q.data_ptr(), n, R.data_ptr(), l)
S = torch.empty(l, l, dtype=torch.float64, device="cuda"); T = torch.empty_like(S); sig = torch.empty(l, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st3 = lib.slra_svd(ctx, R.data_ptr(), l, l, l, S.data_ptr(), l, sig.data_ptr(), T.data_ptr(), l)
e1.record(); torch.cuda.synchronize()
print("status", st, st2, st3, "svd(R) ms", e0.elapsed_time(e1))
print("sigma", sig.cpu().numpy()[[0, 10, 20, 31, 32, 40, 47]])
Rh = R.cpu().numpy().T
import numpy as np
print("numpy sigma", np.linalg.svd(Rh, compute_uv=False)[[0, 10, 20, 31, 32, 40, 47]])
print("R diag", np.diag(Rh)[[0, 10, 20, 31, 32, 40, 47]], "nan?", np.isnan(Rh).any())
