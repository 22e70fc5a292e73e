"""Config-2 range finder, per-family device times with the fused cluster
CholeskyQR3 on and off (SLRA_NO_CLUSTER_CHOLQR). Measurement helper.
usage (GPU box): python tools/cholqr_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1611_01391_b200 as slra  # noqa: E402

st = torch.cuda.Stream()
torch.cuda.set_stream(st)
slra.set_device(0, st.cuda_stream)
work = bench.Config2(slra, torch, 0)
for mode in ("0", "1"):
    os.environ["SLRA_NO_CLUSTER_CHOLQR"] = mode
    for _ in range(5):
        work.step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in ev:
        a.record(st)
        work.step()
        b.record(st)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / len(ev)
    slra.set_timing(True)
    for _ in range(20):
        work.step()
    torch.cuda.synchronize()
    fam = slra.timing_report()
    slra.set_timing(False)
    print(json.dumps({"cluster_cholqr": mode == "0", "ms_per_step": ms, "residual_rel": work.last_residual_rel(),
                      "families_ms_per_step": {k: round(v[0] / 20, 5) for k, v in fam.items()}}))
