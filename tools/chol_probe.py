"""Phase timestamps of the cluster Cholesky (config 4 sketch, both samplers).
usage: LD_LIBRARY_PATH=tools/prof_build/chol/lib python tools/chol_probe.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1611_01391_b200 as slra  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, "tools", "prof_build", "chol", "lib", "libslra_cuda.so"))
rng = np.random.default_rng(1)
m, d, k = 1 << 16, 256, 4096
A = np.asfortranarray(rng.standard_normal((m, d)))
b = A @ rng.standard_normal(d) + 1e-6 * rng.standard_normal(m)
F = slra.make_sub_identity(slra.Rng(3).distinct_indices(k, m), m)
for it in range(3):
    slra.sketch_solve(A, b, F, False)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (8 * 64))()
assert lib.slra_debug_chol_marks(buf) == 0
t = np.array(buf[:], dtype=np.float64).reshape(8, 64)
t0 = t[:, 0][t[:, 0] > 0].min()
for q in range(8):
    row = {i: (t[q, i] - t0) / 1e3 for i in range(64) if t[q, i] > 0}
    print(q, " ".join(f"{i}:{v:.1f}" for i, v in sorted(row.items())))
