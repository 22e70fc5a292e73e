"""Config-2 e2e breakdown: pinned H2D of A alone, the full host-buffer call,
and the host call's parts (python/binding overhead) — run under gpurun."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1611_01391_b200 as slra

c = bench.Config2(slra, torch, 0)
N2 = bench.N2
host = torch.empty(N2 * N2, dtype=torch.float64, pin_memory=True)
host.copy_(c.At.reshape(-1))
dev = torch.empty_like(host, device="cuda")
Hs = [H for _, H in c.ops]
for _ in range(3):
    dev.copy_(host, non_blocking=True)
    slra.range_finder_batched_host(host.data_ptr(), N2, N2, Hs, bench.RANK, True)
torch.cuda.synchronize()
K = 10
t0 = time.perf_counter()
for _ in range(K):
    dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
for _ in range(K):
    slra.range_finder_batched_host(host.data_ptr(), N2, N2, Hs, bench.RANK, True)
torch.cuda.synchronize()
t2 = time.perf_counter()
out = torch.empty(4 * N2 * bench.RANK, dtype=torch.float64)
src = torch.empty(4 * N2 * bench.RANK, dtype=torch.float64, device="cuda")
t3 = time.perf_counter()
for _ in range(K):
    out.copy_(src)
torch.cuda.synchronize()
t4 = time.perf_counter()
print("h2d %.3f ms (%.1f GB/s); host call %.3f ms; 4 MB d2h to pageable %.3f ms" %
      ((t1 - t0) / K * 1e3, 8 * N2 * N2 / ((t1 - t0) / K) / 1e9, (t2 - t1) / K * 1e3, (t4 - t3) / K * 1e3))
slra.set_timing(True)
slra.range_finder_batched_host(host.data_ptr(), N2, N2, Hs, bench.RANK, True)
print(slra.timing_report())
