"""Measure FP64 roofline denominators on the GPU box: cuBLAS DGEMM (via torch) + DMMA/DFMA microbenchmarks."""
import json, subprocess, sys, os, torch
def dgemm(n=8192, reps=10):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2 * n**3 / (best * 1e-3) / 1e12
print(json.dumps({"kind": "cublas_dgemm_8192", "tflops": round(dgemm(), 2), "gpu": torch.cuda.get_device_name()}))
here = os.path.dirname(os.path.abspath(__file__))
print(subprocess.run([os.path.join(here, "fp64_peak")], capture_output=True, text=True).stdout)
