"""Per-phase critical-path cycles of the config-5 C-A block kernel.
usage: LD_LIBRARY_PATH=tools/prof_build/lib python tools/phase_probe.py [blocks]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1611_01391_b200 as slra  # noqa: E402

NAMES = ["init+prefetch", "stage strip", "house_qr", "form_q", "sel argmax", "sel reflector", "sel update",
         "sel backsolve", "sel swaps", "nucleus load", "nucleus jacobi", "nucleus finish", "resid P",
         "resid DMMA", "resid Q"]
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
lib = ctypes.CDLL(os.environ.get("SLRA_PROF_LIB", os.path.join(ROOT, "tools", "prof_build", "lib", "libslra_cuda.so")))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
slra.set_device(0, stream.cuda_stream)


class Comm:
    world, rank = 1, 0


w = bench.Config5(slra, torch, 0, nb, Comm())
w.step()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 32)()
lib.slra_debug_phase_cycles(buf, 32, 1)
w.step()
torch.cuda.synchronize()
lib.slra_debug_phase_cycles(buf, 32, 1)
cyc = np.array(buf[:len(NAMES)], dtype=np.float64) / nb

print(f"nucleus: mean Jacobi sweeps {buf[20] / nb:.2f}, mean kept rows of R {buf[21] / nb:.2f}")
tot = cyc.sum()
print(f"{nb} blocks: {tot:.0f} cycles per block on the critical path")
for n, c in zip(NAMES, cyc):
    print(f"  {n:16s} {c:10.0f}  {100 * c / tot:5.1f}%")
