#!/usr/bin/env python
"""bench.py — BASELINE.json metric "LRA matrix entries/s (sketch+CUR+residual)".

Default workload (N=1 line): config 5 = configs[4] of BASELINE.json, the
largest configuration that fits one GPU (BASELINE's metric names no config):
65,536 independent 256 x 256 fp64 log-kernel blocks K_ij = log|p_i - q_j|
(points uniform in two unit squares 4 apart, seeded per block with the
reference Rng), each factorised by cross_approx (k = l = 32, 2 sweeps, rank
r = numerical_rank(G, 1e-10) adaptive, i.e. the "rank-16 CUR" at its
numerical rank) plus its Frobenius residual ||B - CUR||_F — the per-block
ca_factors -> cross_approx -> cur_evaluate pattern of hss.cpp:47-55 /
cur.cpp:80-82. One step = the whole batch (4.29 G entries, 34.4 GB in HBM).
`--config 1|2|3|4` run the other configurations.

Timing: W untimed warm-up steps, then K steps timed with CUDA events on the
product's stream; an L2 flush (256 MiB write, > 126 MB L2) runs between timed
steps outside the event pairs (config 5's inputs are also 270x the L2);
barrier + synchronize on both sides; the max over ranks. With --gpus N and no
WORLD_SIZE in the environment the script re-launches itself under
torch.distributed.run with N ranks; config 5 then splits the blocks evenly
over the ranks with no communication ("strong": the total work is fixed).

`--impl reference` times the reference algorithm on the host CPU: the C++
oracle restatement (oracle/; the reference itself cannot be built here: no
Eigen) on a bounded sample of the same workload with all host threads, on
the same config/metric/unit. Under torchrun only rank 0 runs it.
"""
import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N2 = 4096
L_SKETCH = 48
RANK = 32


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--blocks", type=int, default=65536, help="config 5 block count")
    p.add_argument("--e2e-steps", type=int, default=5, help="end-to-end (host buffers) steps (config 5)")
    p.add_argument("--ref-blocks", type=int, default=1024, help="config-5 blocks per reference-arm step")
    p.add_argument("--no-other-configs", action="store_true",
                   help="skip the short configs 1-4 legs appended to the default (config 5, N=1) line")
    return p.parse_args()


def maybe_spawn(args):
    """--gpus N without a torchrun environment: re-launch under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------- environment
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() in ("active", "1"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_peaks():
    peaks = {"hbm_gbs": None, "fp64_tflops": None, "fp64_source": None}
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peaks["hbm_gbs"] = mp.get("hbm_gbs")
    except (OSError, ValueError):
        peaks["hbm_gbs"] = 6650.0  # B200_PROFILING.md fallback
    # FP64 is not in MEASURED_PEAKS.json: our DMMA microbenchmark measured on
    # this pool's B200 (profiles/r01_fp64_peaks.jsonl, tools/fp64_peak.cu).
    try:
        best = 0.0
        for line in open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.jsonl")):
            if not line.strip():
                continue
            d = json.loads(line)
            if d.get("kind", "").startswith("dmma"):
                best = max(best, d["tflops"])
        peaks["fp64_tflops"] = best or None
        peaks["fp64_source"] = "profiles/r01_fp64_peaks.jsonl (DMMA microbenchmark, measured)"
    except (OSError, ValueError):
        pass
    return peaks


def profiled_traffic(config, kernel, tag="r01", blocks=None):
    """DRAM bytes (read + write) per launch of `kernel` from the committed
    `ncu --set full` capture (profiles/<tag>_c<config>_traffic.json, written by
    tools/summarize_profiles.py), or None when not captured. Batched captures
    record their block count; the bytes scale to `blocks`."""
    if kernel is None:
        return None
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", f"{tag}_c{config}_traffic.json")))[kernel]
        b = d["dram_bytes"]
        if blocks and d.get("blocks"):
            b *= blocks / d["blocks"]
        return b
    except (OSError, ValueError, KeyError):
        return None


# ---------------------------------------------------------------- config 2 inputs
def config2_matrix_colmajor(seed, device):
    """A = U diag(sigma) V^T with U, V from QR of seeded Gaussians; returns a
    torch tensor holding A in column-major order (i.e. the row-major A^T)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    Gu = torch.randn(N2, N2, dtype=torch.float64, generator=g).to(device)
    Gv = torch.randn(N2, N2, dtype=torch.float64, generator=g).to(device)
    U, Ru = torch.linalg.qr(Gu)
    V, Rv = torch.linalg.qr(Gv)
    U = U * torch.sign(torch.diagonal(Ru))[None, :]
    V = V * torch.sign(torch.diagonal(Rv))[None, :]
    j = torch.arange(N2, dtype=torch.float64, device=device)
    sig = torch.where(j < 32, 0.5 ** j, torch.full_like(j, 1e-12))
    At = (V * sig[None, :]) @ U.T  # = A^T row-major = A column-major
    del Gu, Gv, U, V
    return At.contiguous()


def config2_operators(mod, seed):
    ra = mod.Rng(mod.Rng.derive_seed(seed, 1))
    Ha = mod.take_columns_random(mod.gen_sparse_circulant(N2, 4, ra), L_SKETCH, ra)
    rb = mod.Rng(mod.Rng.derive_seed(seed, 2))
    Hb = mod.take_columns_random(mod.gen_asph(N2, 3, rb), L_SKETCH, rb)
    return [("sparse_pm1_s4", Ha), ("abridged_hadamard_d3", Hb)]


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    if args.config == 5:
        return run_reference_config5(args, ws)
    if args.config != 2:
        print(json.dumps({"impl": "reference", "unavailable": f"reference arm implemented for configs 2 and 5 "
                                                              f"(config {args.config} requested)"}), flush=True)
        return
    import torch  # CPU only: input generation
    sys.path.insert(0, os.path.join(ROOT, "oracle", "build"))
    import _oracle as oracle
    cores = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(cores)
    torch.set_num_threads(cores)
    At = config2_matrix_colmajor(args.seed, "cpu")
    A = At.numpy().T  # column-major view -> (n, n) Fortran array
    ops = config2_operators(oracle, args.seed)

    # each reference step = ONE range-finder LRA + residual (multipliers
    # alternate), i.e. a bounded sample of half a config-2 step: n^2 entries
    def step(i):
        _, H = ops[i % 2]
        U, V = oracle.range_finder(A, H, RANK, True)
        oracle.lowrank_residual_frobenius(A, U, V)

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    dt = time.perf_counter() - t0
    entries = 1.0 * N2 * N2 * args.steps
    value = entries / dt
    line = {
        "impl": "reference", "metric": "LRA matrix entries/s (sketch+CUR+residual)", "value": value,
        "unit": "entries/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, config-2 recipe)",
        "config": {"workload": "config2: range-finder LRA 4096x4096 fp64, l=48, sparse+-1 (s=4) and "
                               "abridged Hadamard (d=3) multipliers, TruncatedRankR r=32, ||A-UV||_F",
                   "entries_per_step": N2 * N2, "m": N2, "n": N2, "l": L_SKETCH, "r": RANK},
        "cpu_baseline": {"value": value, "unit": "entries/s", "cores": cores, "kind": "port",
                         "sample": "per step one config-2 LRA (multipliers alternate; n^2 entries), oracle/ C++ "
                                   "restatement, OpenMP over output columns"},
        "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


C5_M, C5_K, C5_LOOPS = 256, 32, 2
C5_WORKLOAD = ("config5: {blocks} batched 256x256 fp64 log-kernel blocks K_ij = log|p_i - q_j| (points in unit "
               "squares 4 apart, seeded per block), cross_approx k=l=32, 2 sweeps, adaptive r = numerical_rank(G, "
               "1e-10), + per-block ||B - CUR||_F")
# SURVEY.md §8d, config 5, per block: residual 2*256*32*32 + 2*256*32*256 + 3*256^2 = 4.92 MFLOP, four strip
# QRs of ~1 MFLOP; one pass over the block is 256*256*8 bytes
C5_FLOPS_PER_BLOCK = 2.0 * 256 * 32 * 32 + 2.0 * 256 * 32 * 256 + 3.0 * 256 * 256 + 4 * 1.0e6
C5_BYTES_PER_BLOCK = 8.0 * 256 * 256


def config5_host_inputs(mod, seed, b0, nb):
    """Points and initial rows of blocks b0..b0+nb-1 (reference Rng, per-block seeds)."""
    m, k = C5_M, C5_K
    px, py = np.empty((nb, m)), np.empty((nb, m))
    qx, qy = np.empty((nb, m)), np.empty((nb, m))
    init = np.empty((nb, k), dtype=np.int64)
    mod.gen_log_kernel_batch(seed, b0, nb, m, m, k, px.ctypes.data, py.ctypes.data, qx.ctypes.data,
                             qy.ctypes.data, init.ctypes.data)
    return px, py, qx, qy, init


def config5_host_blocks(px, py, qx, qy):
    """Column-major blocks on the host, row-major (nb, n, m) array = each block K^T (numpy's log)."""
    dx = px[:, None, :] - qx[:, :, None]
    dy = py[:, None, :] - qy[:, :, None]
    return 0.5 * np.log(dx * dx + dy * dy)


def oracle_blocks(oracle, blocks, init, threads):
    nb = blocks.shape[0]
    return oracle.cross_approx_blocks(blocks.ctypes.data, nb, C5_M, C5_M, C5_M, C5_M * C5_M, init, C5_K, C5_K,
                                      C5_LOOPS, 1.1, threads)


def run_reference_config5(args, ws):
    """The reference path (oracle/ C++ restatement: cross_approx -> numerical_rank -> primitive_cur ->
    cur_evaluate per block) on the host cores, all threads, each step a bounded sample of the config-5 batch."""
    import paper_1611_01391_b200 as slra  # host-side input generator only (no device work)
    sys.path.insert(0, os.path.join(ROOT, "oracle", "build"))
    import _oracle as oracle
    cores = os.cpu_count() or 1
    nb = min(args.ref_blocks, args.blocks)
    px, py, qx, qy, init = config5_host_inputs(slra, args.seed, 0, nb)
    blocks = np.ascontiguousarray(config5_host_blocks(px, py, qx, qy))
    for _ in range(args.warmup):
        oracle_blocks(oracle, blocks, init, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_blocks(oracle, blocks, init, cores)
    dt = time.perf_counter() - t0
    value = nb * C5_M * C5_M * args.steps / dt
    sample = (f"per step the first {nb} of the {args.blocks} config-5 blocks through the oracle/ C++ restatement of "
              f"the reference path, blocks spread over {cores} OpenMP threads (the reference is single-threaded "
              f"per block)")
    line = {
        "impl": "reference", "metric": "LRA matrix entries/s (sketch+CUR+residual)", "value": value,
        "unit": "entries/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; BASELINE config-5 recipe, reference Rng)",
        "config": config5_config(args.blocks),
        "cpu_baseline": {"value": value, "unit": "entries/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config5_config(blocks):
    return {"workload": C5_WORKLOAD.format(blocks=blocks), "entries_per_step": blocks * C5_M * C5_M,
            "blocks": blocks, "m": C5_M, "n": C5_M, "k": C5_K, "l": C5_K, "loops": C5_LOOPS}


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rc = maybe_spawn(args)
    if rc is not None:
        sys.exit(rc)
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1611_01391_b200 as slra
    # one dedicated stream for the product, the L2 flush and the CUDA events
    # (the legacy default stream has handle 0, which the C-ABI would replace
    # by a private stream)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    slra.set_device(local, stream.cuda_stream)
    peaks = load_peaks()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    flush_buf = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 256 MiB > L2

    from paper_1611_01391_b200 import shard
    comm = shard.Comm(dist)
    if args.config == 2:
        work = Config2(slra, torch, args.seed + rank)
    elif args.config == 3:
        work = Config3(slra, torch, args.seed) if ws == 1 else Config3Sharded(slra, torch, args.seed, comm)
    elif args.config == 4:
        work = Config4(slra, torch, args.seed, comm)
    elif args.config == 1:
        work = Config1(slra, torch, args.seed + rank)
    else:
        work = Config5(slra, torch, args.seed, args.blocks, comm)
    scaling = getattr(work, "scaling", "weak")

    for _ in range(args.warmup):
        work.step()
    barrier()

    # ---- timed region
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = slra.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    for i in range(args.steps):
        flush_buf.fill_(float(i))
        ev[i][0].record(stream)
        work.step()
        ev[i][1].record(stream)
    barrier()
    clocks = sampler.stop()
    gpu_launches = slra.launch_count() - launches0
    ms_total = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # weak: every rank runs its own replica; strong: the ranks share one job
    value = work.entries_per_step * args.steps * (ws if scaling == "weak" else 1) / (ms_max * 1e-3)

    # ---- per-kernel device times over the same K steps (instrumented pass)
    slra.set_timing(True)
    for i in range(args.steps):
        flush_buf.fill_(float(i))
        work.step()
    torch.cuda.synchronize()
    fam = slra.timing_report()
    slra.set_timing(False)
    roofline, kernels = work.roofline(fam, peaks, args.steps)

    # ---- end-to-end through the reference-facing API with host buffers
    e2e = None
    if hasattr(work, "e2e"):
        e2e_steps = args.e2e_steps if args.config == 5 else args.steps
        if e2e_steps > 0 and (ws == 1 or scaling == "weak" or args.config == 5):
            barrier()
            e2e = work.e2e(e2e_steps, args.warmup)
            if e2e is not None and ws > 1 and scaling == "strong":
                # every rank streamed its own share: the job's time is the slowest rank's
                dt = torch.tensor([work.entries_per_step * e2e_steps / ws / e2e["value"]], dtype=torch.float64,
                                  device="cuda")
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
                e2e["value"] = work.entries_per_step * e2e_steps / float(dt.item())
                e2e["h2d_bytes_per_step"] *= ws
                e2e["d2h_bytes_per_step"] *= ws

    line = {
        "metric": "LRA matrix entries/s (sketch+CUR+residual)", "value": value, "unit": "entries/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": getattr(work, "data", "synthetic (seeded; same recipe as BASELINE.json config)"),
        "config": work.config,
        "parallelism": getattr(work, "parallelism", f"replicas x{ws} (no data-path collective)"),
        "l2": "256 MiB flush between timed steps (outside the event pairs)",
        "roofline": roofline, "kernels_ms_per_step": kernels,
        "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clocks,
        "residual_rel": work.last_residual_rel(),
    }
    if hasattr(work, "e2e_dense") and ws == 1 and args.e2e_steps > 0:
        line["e2e_dense_blocks"] = work.e2e_dense(args.e2e_steps, args.warmup)
    if hasattr(work, "function_oracle") and ws == 1 and (args.e2e_steps > 0 or args.config != 5):
        line["function_oracle"] = work.function_oracle(min(args.steps, 10), args.warmup)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = work.cpu_baseline()
    if ws == 1 and args.config == 5 and not args.no_other_configs and args.blocks == 65536:
        # the other BASELINE configs as short legs of the same run (same timing
        # rules: W warm-ups, L2 flush between steps, CUDA events on the product's
        # stream), so the default line carries a measurement of every config
        del work
        gc.collect()
        torch.cuda.empty_cache()
        line["other_configs"] = other_configs(slra, torch, args, comm, stream, flush_buf, peaks)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def other_configs(slra, torch, args, comm, stream, flush_buf, peaks):
    """Configs 1-4 (BASELINE.json configs[0..3]) measured briefly after the
    config-5 line: device-resident entries/s, the per-kernel family times, the
    dominant kernel's roofline and the host-buffer e2e; no CPU baseline."""
    out = {}
    steps, warmup = 10, max(3, min(args.warmup, 5))
    makers = {
        "config1": lambda: Config1(slra, torch, args.seed),
        "config2": lambda: Config2(slra, torch, args.seed),
        "config3": lambda: Config3(slra, torch, args.seed),
        "config4": lambda: Config4(slra, torch, args.seed, comm),
    }
    for name, make in makers.items():
        try:
            work = make()
            for _ in range(warmup):
                work.step()
            torch.cuda.synchronize()
            launches0 = slra.launch_count()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for i in range(steps):
                flush_buf.fill_(float(i))
                ev[i][0].record(stream)
                work.step()
                ev[i][1].record(stream)
            torch.cuda.synchronize()
            launches = slra.launch_count() - launches0
            ms = sum(a.elapsed_time(b) for a, b in ev) / steps
            slra.set_timing(True)
            for i in range(steps):
                flush_buf.fill_(float(i))
                work.step()
            torch.cuda.synchronize()
            fam = slra.timing_report()
            slra.set_timing(False)
            roofline, kernels = work.roofline(fam, peaks, steps)
            e2e = work.e2e(steps, warmup)
            out[name] = {
                "workload": work.config.get("workload"), "entries_per_step": work.entries_per_step,
                "value": work.entries_per_step / (ms * 1e-3), "unit": "entries/s", "ms_per_step": ms,
                "steps": steps, "warmup": warmup, "gpu_launches": launches,
                "roofline": roofline, "kernels_ms_per_step": kernels, "e2e": e2e,
                "residual_rel": work.last_residual_rel(),
            }
            del work
        except Exception as exc:  # a failed leg must not lose the headline line
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
        gc.collect()
        torch.cuda.empty_cache()
    return out


class Config2:
    def __init__(self, slra, torch, seed):
        self.slra, self.torch = slra, torch
        self.seed = seed
        self.At = config2_matrix_colmajor(seed, "cuda")
        self.ops = config2_operators(slra, seed)
        self.plans = []
        for name, H in self.ops:
            p = H.plan("right")
            dev = dict(src=torch.tensor(p["src"], dtype=torch.int64, device="cuda"),
                       coef=torch.tensor(p["coef"], dtype=torch.float64, device="cuda"),
                       q=torch.tensor(p["q"], dtype=torch.int32, device="cuda"))
            self.plans.append((name, p, dev))
        self.U = [torch.empty(RANK, N2, dtype=torch.float64, device="cuda") for _ in self.ops]  # col-major m x r
        self.V = [torch.empty(N2, RANK, dtype=torch.float64, device="cuda") for _ in self.ops]  # col-major r x n
        self.out = torch.zeros(len(self.ops), 2, dtype=torch.float64, device="cuda")
        self.entries_per_step = 2 * N2 * N2
        self.config = {"workload": "config2: range-finder LRA 4096x4096 fp64, l=48, sparse+-1 (s=4) and "
                                   "abridged Hadamard (d=3) multipliers, TruncatedRankR r=32, ||A-UV||_F",
                       "entries_per_step": self.entries_per_step, "m": N2, "n": N2, "l": L_SKETCH, "r": RANK}

    def step(self):
        # both multipliers in one call: their TSQR/SVD stages run concurrently
        plans = [(p["width"], p["tree"], d["src"].data_ptr(), d["coef"].data_ptr(), d["q"].data_ptr())
                 for _, p, d in self.plans]
        self.slra.range_finder_batched_device(self.At.data_ptr(), N2, N2, N2, plans, L_SKETCH, RANK, True,
                                              [u.data_ptr() for u in self.U], N2,
                                              [v.data_ptr() for v in self.V], RANK, self.out.data_ptr())

    def last_residual_rel(self):
        o = self.out.cpu().numpy()
        return {name: float((o[i, 0] / o[i, 1]) ** 0.5) for i, (name, _, _) in enumerate(self.plans)}

    def roofline(self, fam, peaks, steps):
        m = n = N2
        kernels = {k: v[0] / steps for k, v in fam.items()}
        # dominant family by device time
        top = max(fam.items(), key=lambda kv: kv[1][0])[0]
        per_launch_ms = {k: v[0] / max(v[1], 1) for k, v in fam.items()}
        if top in ("residual", "gemm_v"):
            flops = 2.0 * m * n * RANK + (5.0 * m * n if top == "residual" else 0.0)
            ach = flops / (per_launch_ms[top] * 1e-3) / 1e12
            rl = {"kernel": top, "bound": "tensor", "achieved": ach, "peak": peaks["fp64_tflops"],
                  "unit": "TFLOP/s", "frac": ach / peaks["fp64_tflops"] if peaks["fp64_tflops"] else None,
                  "peak_source": peaks["fp64_source"],
                  "algorithmic_per_launch": {"flops": flops, "bytes": 8.0 * m * n + 16.0 * m * RANK},
                  "traffic": None}
        else:
            # latency-bound small dense factorisations (the 48 x 48 Jacobi SVD,
            # the CholeskyQR steps): algorithmic bytes = the operands they read
            # and write once (l x l per sketch for svd; the sketch strip for QR)
            byts = {"sketch": 8.0 * m * L_SKETCH * (4 + 8) / 2 + 8.0 * m * L_SKETCH,
                    "svd": 2 * 4 * 8.0 * L_SKETCH * L_SKETCH}.get(top, 8.0 * m * L_SKETCH)
            ach = byts / (per_launch_ms[top] * 1e-3) / 1e9
            rl = {"kernel": top, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                  "frac": ach / peaks["hbm_gbs"], "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                  "algorithmic_bytes_per_launch": byts,
                  "traffic": profiled_traffic(2, {"svd": "svd_cta_kernel"}.get(top), tag="r02"),
                  "note": "latency-bound: one CTA per sketch runs a serial chain (Jacobi rounds, FP64 FMA "
                          "latency ~24 cycles); see kernels_ms_per_step and profiles/"}
        # the HBM/FP64-tensor kernels on their own rooflines, always reported
        if "residual" in fam:
            flops = 2.0 * m * n * RANK + 5.0 * m * n
            ach = flops / (per_launch_ms["residual"] * 1e-3) / 1e12
            rl["residual_kernel"] = {"achieved_tflops": ach, "frac_fp64": ach / peaks["fp64_tflops"],
                                     "achieved_gbs": 8.0 * m * n / (per_launch_ms["residual"] * 1e-3) / 1e9,
                                     "traffic": profiled_traffic(2, "residual_stream_kernel", tag="r02")}
        if "gemm_v" in fam:
            flops = 2.0 * m * n * RANK
            ach = flops / (per_launch_ms["gemm_v"] * 1e-3) / 1e12
            rl["gemm_v_kernel"] = {"achieved_tflops": ach, "frac_fp64": ach / peaks["fp64_tflops"],
                                   "achieved_gbs": 8.0 * m * n / (per_launch_ms["gemm_v"] * 1e-3) / 1e9,
                                   "traffic": profiled_traffic(2, "tn_skinny_kernel", tag="r02")}
        return rl, kernels

    def e2e(self, steps, warmup):
        torch = self.torch
        host = torch.empty(N2 * N2, dtype=torch.float64, pin_memory=True)
        host.copy_(self.At.reshape(-1))
        ptr = host.data_ptr()
        ops = self.ops

        Hs = [H for _, H in ops]

        def one():
            # both multipliers of the step on one upload of A (the batched
            # form of range_finder(M, H, r, TruncatedRankR))
            self.slra.range_finder_batched_host(ptr, N2, N2, Hs, RANK, True)
        for _ in range(max(1, warmup // 2)):
            one()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        return {"value": self.entries_per_step * steps / dt, "unit": "entries/s",
                "h2d_bytes_per_step": 8 * N2 * N2 + sum(8 * 2 * L_SKETCH * 8 + 4 * L_SKETCH for _ in Hs),
                "d2h_bytes_per_step": 2 * (8 * 2 * N2 * RANK + 16),
                "api": "paper_1611_01391_b200.range_finder_batched_host -> slra_range_finder_batched "
                       "(host pinned A in once, both multipliers' plans, U/V and residuals out)"}

    def cpu_baseline(self):
        sys.path.insert(0, os.path.join(ROOT, "oracle", "build"))
        import _oracle as oracle
        cores = os.cpu_count() or 1
        A = self.At.cpu().numpy().T
        ops = config2_operators(oracle, self.seed)
        t0 = time.perf_counter()
        for _, H in ops:
            U, V = oracle.range_finder(A, H, RANK, True)
            oracle.lowrank_residual_frobenius(A, U, V)
        dt = time.perf_counter() - t0
        return {"value": self.entries_per_step / dt, "unit": "entries/s", "cores": cores, "kind": "port",
                "sample": "one full config-2 step (both multipliers on the same 4096^2 A) through the oracle/ "
                          "C++ restatement of the reference path (full-operator sketch application, pinv via SVD, "
                          "Frobenius residual), OpenMP over output columns", "seconds": dt}


class Config1:
    """Config 1: 256x256 factor-Gaussian CUR, 3 C-A sweeps + residual (latency-bound)."""

    def __init__(self, slra, torch, seed):
        self.slra, self.torch = slra, torch
        A = slra.gen_factor_gaussian(256, 256, 8, 1e-8, slra.Rng(seed))
        self.A_host = A
        self.A = torch.from_numpy(A.T.copy()).cuda()
        self.init = torch.tensor(slra.Rng(seed + 1).distinct_indices(16, 256), dtype=torch.int64, device="cuda")
        self.I = torch.zeros(16, dtype=torch.int64, device="cuda")
        self.J = torch.zeros(16, dtype=torch.int64, device="cuda")
        self.U = torch.zeros(256, dtype=torch.float64, device="cuda")
        self.entries_per_step = 256 * 256
        self.config = {"workload": "config1: C-A CUR 256x256, r=8, k=l=16, 3 sweeps, Frobenius residual",
                       "entries_per_step": self.entries_per_step}
        self.res = (0.0, 1.0)

    def step(self):
        s = self.slra
        s.cross_approx_device(self.A.data_ptr(), 256, 256, 256, 8, 16, 16, self.init.data_ptr(), 3, 1.1,
                              self.I.data_ptr(), self.J.data_ptr(), self.U.data_ptr())
        self.res = s.cur_residual_device(self.A.data_ptr(), 256, 256, 256, self.I.data_ptr(), 16,
                                         self.J.data_ptr(), 16, self.U.data_ptr())

    def last_residual_rel(self):
        return (self.res[0] / self.res[1]) ** 0.5

    def roofline(self, fam, peaks, steps):
        kernels = {k: v[0] / steps for k, v in fam.items()}
        top = max(fam.items(), key=lambda kv: kv[1][0])[0]
        per = fam[top][0] / max(fam[top][1], 1)
        # 2*256*16*16 + 2*256*16*256 + 3*256^2 ~ 2.42 MFLOP, ~11 B per entry
        flops = 2.0 * 256 * 16 * 16 + 2.0 * 256 * 16 * 256 + 3.0 * 256 * 256
        ach = flops / (per * 1e-3) / 1e12
        return {"kernel": top, "bound": "tensor", "achieved": ach, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                "frac": ach / peaks["fp64_tflops"] if peaks["fp64_tflops"] else None,
                "peak_source": peaks["fp64_source"], "algorithmic_per_launch": {"flops": flops},
                "traffic": profiled_traffic(1, "ca_block_kernel", tag="r02"),
                "note": "config 1 is one 256x256 problem: one CTA's dependent chain (launch/latency bound, "
                        "SURVEY 8d); the FP64 fraction is reported for completeness"}, kernels

    def e2e(self, steps, warmup):
        s = self.slra

        def one():
            g = s.cross_approx(self.A_host, 8, 16, 16, [], 3, 1.1, s.Rng(1))
            s.cur_evaluate(self.A_host, g["I"], g["J"], g["nucleus"])
        for _ in range(max(1, warmup // 2)):  # first-use costs (pool growth, attributes) stay out
            one()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        dt = time.perf_counter() - t0
        return {"value": self.entries_per_step * steps / dt, "unit": "entries/s",
                "h2d_bytes_per_step": 2 * 8 * 256 * 256, "d2h_bytes_per_step": 8 * (16 + 16 + 256)}

    def cpu_baseline(self):
        sys.path.insert(0, os.path.join(ROOT, "oracle", "build"))
        import _oracle as oracle
        n = 0
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 5.0:
            o = oracle.cross_approx(self.A_host, 8, 16, 16, [], 3, 1.1, None, oracle.Rng(n))
            oracle.cur_evaluate(self.A_host, o["I"], o["J"], o["nucleus"])
            n += 1
        dt = time.perf_counter() - t0
        return {"value": self.entries_per_step * n / dt, "unit": "entries/s", "cores": 1, "kind": "port",
                "sample": f"{n} config-1 runs in 5 s"}


N3, K3, LOOPS3 = 16384, 64, 5


def config3_points(mod, seed, n=N3):
    """x_i ~ U[0,1], y_j ~ U[2,3] drawn with the reference Rng (testgen order)."""
    r = mod.Rng(seed)
    x = [r.uniform() for _ in range(n)]
    y = [2.0 + r.uniform() for _ in range(n)]
    return x, y


class Config3:
    """Config 3: C-A on the 16384^2 Cauchy block 1/(x_i - y_j), k=l=64, 5 sweeps,
    adaptive r (numerical_rank 1e-10), full ||A - CUR||_F."""

    def __init__(self, slra, torch, seed):
        self.slra, self.torch = slra, torch
        self.seed = seed
        x, y = config3_points(slra, seed)
        xd = torch.tensor(x, dtype=torch.float64, device="cuda")
        yd = torch.tensor(y, dtype=torch.float64, device="cuda")
        # column-major A: At[j, i] = 1/(x_i - y_j) (one IEEE division: bit-identical to the host generator)
        self.At = (1.0 / (xd[None, :] - yd[:, None])).contiguous()
        self.init = slra.Rng(seed + 1).distinct_indices(K3, N3)
        self.init_d = torch.tensor(self.init, dtype=torch.int64, device="cuda")
        self.I = torch.zeros(K3, dtype=torch.int64, device="cuda")
        self.J = torch.zeros(K3, dtype=torch.int64, device="cuda")
        self.U = torch.zeros(K3 * K3, dtype=torch.float64, device="cuda")
        self.T = torch.zeros(K3 * K3, dtype=torch.float64, device="cuda")
        self.S = torch.zeros(K3 * K3, dtype=torch.float64, device="cuda")
        self.out = torch.zeros(2, dtype=torch.float64, device="cuda")
        self.r = 0
        self.entries_per_step = N3 * N3
        self.config = {"workload": "config3: C-A CUR of the 16384x16384 fp64 Cauchy block 1/(x-y), k=l=64, "
                                   "5 sweeps, adaptive r (numerical_rank 1e-10), full ||A-CUR||_F",
                       "entries_per_step": self.entries_per_step, "m": N3, "n": N3, "k": K3, "l": K3,
                       "loops": LOOPS3}

    def step(self):
        s = self.slra
        a = self.At.data_ptr()
        self.r = s.cross_approx_device(a, N3, N3, N3, 0, K3, K3, self.init_d.data_ptr(), LOOPS3, 1.1,
                                       self.I.data_ptr(), self.J.data_ptr(), self.U.data_ptr(),
                                       self.T.data_ptr(), self.S.data_ptr())
        s.cur_residual_factored_device(a, N3, N3, N3, self.I.data_ptr(), K3, self.J.data_ptr(), K3,
                                       self.T.data_ptr(), self.S.data_ptr(), self.r, self.out.data_ptr())

    def last_residual_rel(self):
        o = self.out.cpu().numpy()
        return {"rel": float((o[0] / o[1]) ** 0.5), "r": int(self.r)}

    def roofline(self, fam, peaks, steps):
        kernels = {k: v[0] / steps for k, v in fam.items()}
        per = {k: v[0] / max(v[1], 1) for k, v in fam.items()}
        top = max(fam.items(), key=lambda kv: kv[1][0])[0]
        n, r = N3, max(self.r, 1)
        # algorithmic bytes per launch of each family (DESIGN.md roofline table)
        strip = 8.0 * n * K3
        byts = {"residual": 8.0 * n * n + 16.0 * n * r, "gather": strip * 2, "thin_qr": strip * 2,
                "maxvol": strip}
        b = byts.get(top, strip)
        ach = b / (per[top] * 1e-3) / 1e9
        rl = {"kernel": top, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
              "frac": ach / peaks["hbm_gbs"], "peak_source": "MEASURED_PEAKS.json hbm_gbs",
              "algorithmic_bytes_per_launch": b,
              "traffic": profiled_traffic(3, {"thin_qr": "tsqr_top_kernel", "maxvol": "maxvol_large_kernel",
                                              "residual": "residual_stream_kernel"}.get(top), tag="r02")}
        if "residual" in per:
            rb = 8.0 * n * n + 16.0 * n * r
            rl["residual_kernel"] = {"achieved_gbs": rb / (per["residual"] * 1e-3) / 1e9,
                                     "frac_hbm": rb / (per["residual"] * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                     "inner_dim_r": r}
        return rl, kernels

    def e2e(self, steps, warmup):
        torch = self.torch
        host = torch.empty(N3 * N3, dtype=torch.float64, pin_memory=True)
        host.copy_(self.At.reshape(-1))
        ptr = host.data_ptr()

        def one():
            return self.slra.cross_approx_host(ptr, N3, N3, 0, K3, K3, self.init, LOOPS3, 1.1)
        for _ in range(max(1, warmup // 2)):
            one()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            d = one()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        return {"value": self.entries_per_step * steps / dt, "unit": "entries/s",
                "h2d_bytes_per_step": 8 * N3 * N3 + 8 * K3,
                "d2h_bytes_per_step": 8 * (2 * K3 + K3 * K3 + 2 * K3 * d["r"] + 2),
                "api": "paper_1611_01391_b200.cross_approx_host -> slra::cross_approx + slra::cur_evaluate "
                       "(host pinned A in; I, J, nucleus, residual out)"}

    def function_oracle(self, steps, warmup):
        """The same step with A given by its points (FunctionOracle, oracle.hpp:43-54):
        slra_cross_approx_cauchy + slra_cur_residual_factored_cauchy evaluate the strips, the
        generator and the residual pass's tiles instead of reading the materialised 2 GiB matrix
        (bit-identical results, checked). Device-resident points (CUDA events), then end to end:
        pinned host points in, I, J, nucleus factors and the residual pair out (wall clock)."""
        torch, slra = self.torch, self.slra
        x, y = config3_points(slra, self.seed)
        xd = torch.tensor(x, dtype=torch.float64, device="cuda")
        yd = torch.tensor(y, dtype=torch.float64, device="cuda")
        o = {k: torch.zeros_like(v) for k, v in (("I", self.I), ("J", self.J), ("U", self.U), ("T", self.T),
                                                  ("S", self.S), ("out", self.out))}

        def dev(xp, yp):
            r = slra.cross_approx_cauchy_device(xp, yp, N3, N3, 0, K3, K3, self.init_d.data_ptr(), LOOPS3, 1.1,
                                                o["I"].data_ptr(), o["J"].data_ptr(), o["U"].data_ptr(),
                                                o["T"].data_ptr(), o["S"].data_ptr())
            slra.cur_residual_factored_cauchy_device(xp, yp, N3, N3, o["I"].data_ptr(), K3, o["J"].data_ptr(), K3,
                                                     o["T"].data_ptr(), o["S"].data_ptr(), r, o["out"].data_ptr())
            return r
        for _ in range(max(warmup, 1)):
            dev(xd.data_ptr(), yd.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            r = dev(xd.data_ptr(), yd.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        same = r == self.r and all(bool(torch.equal(o[k], v)) for k, v in (("I", self.I), ("J", self.J),
                                                                          ("U", self.U), ("out", self.out)))
        hx = torch.tensor(x, dtype=torch.float64).pin_memory()
        hy = torch.tensor(y, dtype=torch.float64).pin_memory()
        hout = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in o.items()}

        def e2e_one():
            xs, ys = hx.to("cuda", non_blocking=True), hy.to("cuda", non_blocking=True)
            rr = dev(xs.data_ptr(), ys.data_ptr())
            for k in ("I", "J", "U", "out"):
                hout[k].copy_(o[k], non_blocking=True)
            n_r = K3 * rr
            hout["T"][:n_r].copy_(o["T"][:n_r], non_blocking=True)
            hout["S"][:n_r].copy_(o["S"][:n_r], non_blocking=True)
            torch.cuda.synchronize()
            return rr
        e2e_one()
        t0 = time.perf_counter()
        for _ in range(steps):
            rr = e2e_one()
        dt = time.perf_counter() - t0
        return {"value": self.entries_per_step / (ms * 1e-3), "unit": "entries/s", "ms_per_step": ms,
                "steps": steps, "identical_to_dense_run": same,
                "e2e": {"value": self.entries_per_step * steps / dt, "unit": "entries/s",
                        "h2d_bytes_per_step": 16 * N3, "d2h_bytes_per_step": 8 * (2 * K3 + K3 * K3 + 2 * K3 * rr + 2),
                        "steps": steps},
                "api": "paper_1611_01391_b200.cross_approx_cauchy_device + cur_residual_factored_cauchy_device -> "
                       "slra_cross_approx_cauchy / slra_cur_residual_factored_cauchy (points in; A never "
                       "materialised)"}

    def cpu_baseline(self):
        sys.path.insert(0, os.path.join(ROOT, "oracle", "build"))
        import _oracle as oracle
        cores = os.cpu_count() or 1
        A = self.At.cpu().numpy().T
        t0 = time.perf_counter()
        o = oracle.cross_approx(A, 1, K3, K3, self.init, LOOPS3, 1.1, None, oracle.Rng(0))
        G = A[np.ix_(o["I"], o["J"])]
        rk = oracle.numerical_rank(G, 1e-10, True)
        c = oracle.primitive_cur(A, o["I"], o["J"], rk)
        oracle.cur_evaluate(A, o["I"], o["J"], c["nucleus"])
        dt = time.perf_counter() - t0
        return {"value": self.entries_per_step / dt, "unit": "entries/s", "cores": cores, "kind": "port",
                "sample": "one full config-3 step (5 C-A sweeps on 16384^2, adaptive-rank nucleus, "
                          "cur_evaluate) through the oracle/ C++ restatement, OpenMP", "seconds": dt}


class Config3Sharded:
    """Config 3 row-sharded over the torchrun ranks (shard.cross_approx): total
    work fixed (16384^2), each rank holds m/N rows -> scaling "strong"."""

    scaling = "strong"

    def __init__(self, slra, torch, seed, comm):
        from paper_1611_01391_b200 import shard
        self.slra, self.torch, self.shard, self.comm = slra, torch, shard, comm
        x, y = config3_points(slra, seed)
        self.row0, self.mloc = shard.split(N3, comm.world, comm.rank)
        xd = torch.tensor(x[self.row0:self.row0 + self.mloc], dtype=torch.float64, device="cuda")
        yd = torch.tensor(y, dtype=torch.float64, device="cuda")
        self.At = (1.0 / (xd[None, :] - yd[:, None])).contiguous()  # (n, m_local): local rows, column-major
        self.init = slra.Rng(seed + 1).distinct_indices(K3, N3)
        self.ops = shard.DeviceOps(slra, torch)
        self.res = None
        self.entries_per_step = N3 * N3
        self.parallelism = f"row-sharded x{comm.world}: allreduce(A(I,:)) + allgather(A(:,J)) per sweep, " \
                           f"allreduce of the residual partials (NCCL)"
        self.config = {"workload": "config3: C-A CUR of the 16384x16384 fp64 Cauchy block 1/(x-y), k=l=64, "
                                   "5 sweeps, adaptive r, full ||A-CUR||_F, row-sharded",
                       "entries_per_step": self.entries_per_step, "m": N3, "n": N3, "k": K3, "l": K3,
                       "loops": LOOPS3, "rows_per_rank": self.mloc}

    def step(self):
        self.res = self.shard.cross_approx(self.ops, self.comm, self.At, self.row0, N3, 0, K3, K3, self.init,
                                           LOOPS3, 1.1, self.torch)

    def last_residual_rel(self):
        return {"rel": (self.res.resid_sq / self.res.norm_sq) ** 0.5, "r": self.res.r}

    def roofline(self, fam, peaks, steps):
        return Config3.roofline(self, fam, peaks, steps)

    @property
    def r(self):
        return self.res.r if self.res else 1

    def e2e(self, steps, warmup):
        return None

    def cpu_baseline(self):
        return None


M4, D4, K4 = 1 << 20, 256, 4096


class Config4:
    """Config 4: sketched LSR, A 2^20 x 256 Gaussian, b = A x0 + 1e-6 e; 4096
    rows sampled (a) uniformly, (b) by a sparse +-1 sketch with 2 nonzeros
    per row; solve + ||A x_hat - b||. One step = both samplers (2 x m(d+1)
    entries). N > 1: rows sharded, one allreduce of the sketch (shard.py)."""

    CHUNK = 4096

    def __init__(self, slra, torch, seed, comm):
        from paper_1611_01391_b200 import shard
        self.slra, self.torch, self.shard, self.comm = slra, torch, shard, comm
        ws = comm.world
        self.scaling = "weak" if ws == 1 else "strong"
        self.row0, self.mloc = shard.split(M4, ws, comm.rank)
        # the reference generator (gen_lsr_family pattern, testgen.cpp:159-193,
        # noise 1e-6): A column-major Gaussian, x0, e from one Rng stream —
        # the inputs tests/test_gpu_config4.py checks against the oracle. The
        # stream is sequential, so every rank draws the whole A and keeps its rows.
        A_h, b_h = slra.gen_lsr_gaussian(M4, D4, 1e-6, slra.Rng(2024 + seed))
        self.At = torch.from_numpy(np.ascontiguousarray(A_h[self.row0:self.row0 + self.mloc].T)).cuda()
        self.b = torch.from_numpy(np.ascontiguousarray(b_h[self.row0:self.row0 + self.mloc])).cuda()
        del A_h, b_h
        ru = slra.Rng(slra.Rng.derive_seed(seed, 41))
        Fu = slra.make_sub_identity(ru.distinct_indices(K4, M4), M4)
        rs = slra.Rng(slra.Rng.derive_seed(seed, 42))
        Fs = slra.make_product([slra.make_sub_identity(rs.distinct_indices(K4, M4), M4),
                                slra.gen_sparse_circulant(M4, 2, rs), slra.gen_sign_diagonal(M4, rs)])
        self.ops_host = [("uniform_rows", Fu), ("sparse_pm1_s2", Fs)]
        self.plans = []
        for name, F in self.ops_host:
            p = F.plan("left")
            self.plans.append((name, p, dict(src=torch.tensor(p["src"], dtype=torch.int64, device="cuda"),
                                              coef=torch.tensor(p["coef"], dtype=torch.float64, device="cuda"),
                                              q=torch.tensor(p["q"], dtype=torch.int32, device="cuda"))))
        # both samplers' solutions side by side (D4 x 2, column-major): one
        # residual pass over A certifies both (slra_lsr_residual_multi)
        self.X = torch.zeros(len(self.plans), D4, dtype=torch.float64, device="cuda")
        self.x = [self.X[i] for i in range(len(self.plans))]
        self.out = torch.zeros(len(self.plans), 2, dtype=torch.float64, device="cuda")
        self.sres = [0.0] * len(self.plans)
        self.tres = [0.0] * len(self.plans)
        self.dev_ops = shard.DeviceOps(slra, torch)
        self.entries_per_step = 2 * M4 * (D4 + 1)
        self.data = "synthetic (seeded; reference generator gen_lsr_gaussian, noise 1e-6)"
        if ws > 1:
            self.parallelism = f"row-sharded x{ws}: per-rank sketch contributions + one allreduce (NCCL)"
        self.config = {"workload": "config4: sketched LSR, A 1048576x256 fp64 Gaussian, b = A x0 + 1e-6 e, "
                                   "4096 rows: uniform sampling and sparse +-1 (s=2); solve + ||A x - b||",
                       "entries_per_step": self.entries_per_step, "m": M4, "d": D4, "k": K4,
                       "rows_per_rank": self.mloc}

    def step(self):
        s = self.slra
        if self.comm.world == 1:
            # both samplers' solves side by side (slra_sketch_solve_batched: a cluster per sketch)
            self.sres = s.sketch_solve_batched_device(
                self.At.data_ptr(), M4, M4, D4, self.b.data_ptr(), [d["src"].data_ptr() for _, _, d in self.plans],
                [d["coef"].data_ptr() for _, _, d in self.plans], [d["q"].data_ptr() for _, _, d in self.plans],
                [p["width"] for _, p, _ in self.plans], [p["tree"] for _, p, _ in self.plans], K4,
                [x.data_ptr() for x in self.x])
            # residual_norm of both solutions in ONE pass over A (out[i, 0])
            s.lsr_residual_multi_device(self.At.data_ptr(), M4, M4, D4, self.b.data_ptr(), self.X.data_ptr(),
                                        len(self.plans), self.out.data_ptr())
        else:
            for i, (_, p, d) in enumerate(self.plans):
                x, self.sres[i], self.tres[i] = self.shard.sketch_solve(
                    self.dev_ops, self.comm, self.At, self.b, self.row0, D4, d["src"], d["coef"], p["width"], K4,
                    self.torch)
                self.x[i] = x

    def last_residual_rel(self):
        torch = self.torch
        bn = self.b.norm().item()
        out = {}
        for i, (name, _, _) in enumerate(self.plans):
            tres = self.out.view(-1)[i].item() ** 0.5 if self.comm.world == 1 else self.tres[i]
            out[name] = {"sketched_residual": self.sres[i], "true_residual": tres, "rel_to_b": tres / bn}
        if self.comm.world == 1:
            # residual ratio against the exact LS solution (certification, untimed)
            src = torch.arange(M4, dtype=torch.int64, device="cuda")
            coef = torch.ones(M4, dtype=torch.float64, device="cuda")
            q = torch.zeros(M4, dtype=torch.int32, device="cuda")
            xe = torch.zeros(D4, dtype=torch.float64, device="cuda")
            self.slra.sketch_solve_device(self.At.data_ptr(), M4, M4, D4, self.b.data_ptr(), src.data_ptr(),
                                          coef.data_ptr(), q.data_ptr(), 1, 0, M4, xe.data_ptr())
            o = torch.zeros(2, dtype=torch.float64, device="cuda")
            self.slra.lsr_residual_device(self.At.data_ptr(), M4, M4, D4, self.b.data_ptr(), xe.data_ptr(),
                                          o.data_ptr())
            opt = o[0].item() ** 0.5
            for name in out:
                out[name]["ratio_vs_exact"] = out[name]["true_residual"] / opt
        return out

    def roofline(self, fam, peaks, steps):
        kernels = {k: v[0] / steps for k, v in fam.items()}
        per = {k: v[0] / max(v[1], 1) for k, v in fam.items()}
        top = max(fam.items(), key=lambda kv: kv[1][0])[0]
        # algorithmic bytes per launch: the residual pass reads A|b once; the
        # solve family (Cholesky, triangular solves, sketched residual) reads
        # the k x (d+1) sketch about twice
        byts = {"lsr_residual": 8.0 * self.mloc * (D4 + 1), "sketch": 8.0 * K4 * 2 * (D4 + 1) * 1.5,
                "gemm": 8.0 * K4 * (D4 + 1), "lsr_solve": 2 * 8.0 * K4 * (D4 + 1)}
        b = byts.get(top, 8.0 * self.mloc * (D4 + 1))
        ach = b / (per[top] * 1e-3) / 1e9
        rl = {"kernel": top, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
              "frac": ach / peaks["hbm_gbs"], "peak_source": "MEASURED_PEAKS.json hbm_gbs",
              "algorithmic_bytes_per_launch": b, "traffic": profiled_traffic(4, {"lsr_residual": "lsr_residual_kernel", "lsr_solve": "chol_cluster_kernel"}.get(top), tag="r02")}
        if top == "lsr_solve":
            rl["note"] = ("latency-bound: the 256 x 256 Cholesky, solves and refinement run on one 8-CTA cluster "
                          "(FP64 dependent chains); per-launch mean over the family's kernels")
        else:
            rl["note"] = ("one pass over A|b certifies both samplers' solutions (slra_lsr_residual_multi); "
                          "the solve (Gram on DMMA + 8-CTA cluster Cholesky/solve/refinement) is "
                          f"{kernels.get('lsr_solve', 0.0) + kernels.get('gemm', 0.0) + kernels.get('gemm_reduce', 0.0):.3f} ms/step")
        if "lsr_residual" in per:
            rb = 8.0 * self.mloc * (D4 + 1)
            rl["lsr_residual_kernel"] = {"achieved_gbs": rb / (per["lsr_residual"] * 1e-3) / 1e9,
                                         "frac_hbm": rb / (per["lsr_residual"] * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                         "traffic": profiled_traffic(4, "lsr_residual_kernel", tag="r02")}
        return rl, kernels

    def e2e(self, steps, warmup):
        torch = self.torch
        Ah = torch.empty(M4 * D4, dtype=torch.float64, pin_memory=True)
        Ah.copy_(self.At.reshape(-1))
        bh = torch.empty(M4, dtype=torch.float64, pin_memory=True)
        bh.copy_(self.b)

        def one():
            for _, F in self.ops_host:
                self.slra.sketch_solve_host(Ah.data_ptr(), bh.data_ptr(), M4, D4, F)
        one()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        return {"value": self.entries_per_step * steps / dt, "unit": "entries/s",
                "h2d_bytes_per_step": 2 * 8 * M4 * (D4 + 1), "d2h_bytes_per_step": 2 * 8 * (D4 + 2),
                "api": "paper_1611_01391_b200.sketch_solve_host -> slra_sketch_solve + slra_lsr_residual "
                       "(host pinned A|b in, x_hat and residuals out, once per sampler)"}

    def cpu_baseline(self):
        sys.path.insert(0, os.path.join(ROOT, "oracle", "build"))
        import _oracle as oracle
        cores = os.cpu_count() or 1
        A = self.At.cpu().numpy().T  # (m, d) Fortran
        b = self.b.cpu().numpy()
        ru = oracle.Rng(oracle.Rng.derive_seed(0, 41))
        F = oracle.make_sub_identity(ru.distinct_indices(K4, M4), M4)
        t0 = time.perf_counter()
        rep = oracle.sketch_solve(A, b, F, False)
        oracle.residual_norm(A, b, rep["x_hat"])
        dt = time.perf_counter() - t0
        return {"value": M4 * (D4 + 1) / dt, "unit": "entries/s", "cores": cores, "kind": "port",
                "sample": "one config-4 sampler (uniform rows): oracle sketch_solve (ColPivHouseholderQR of "
                          "the 4096x256 sketch) + residual_norm over the full A", "seconds": dt}


class Config5:
    """Config 5: batched superfast-multipole LRA — 65,536 independent 256 x 256 log-kernel blocks,
    cross_approx k = l = 32, 2 sweeps, adaptive r, fused per-block residual. N ranks split the
    blocks evenly (no communication)."""

    CHUNK = 4096

    def __init__(self, slra, torch, seed, blocks, comm):
        from paper_1611_01391_b200 import shard
        self.slra, self.torch, self.seed, self.blocks = slra, torch, seed, blocks
        ws = comm.world
        self.b0, self.nb = shard.split(blocks, ws, comm.rank)
        self.scaling = "weak" if ws == 1 else "strong"
        self.parallelism = f"block-split x{ws}: {self.nb} blocks per rank, no communication"
        m, nb = C5_M, self.nb
        # inputs: per-block points + initial rows from the reference Rng (host, the
        # same recipe as the oracle/tests), blocks materialised on the device
        self.A = torch.empty(nb, m, m, dtype=torch.float64, device="cuda")
        self.init = torch.empty(nb, C5_K, dtype=torch.int64, device="cuda")
        # the points too (px, py, qx, qy: nb x m each): the FunctionOracle form of the same blocks
        self.pts = torch.empty(4, nb, m, dtype=torch.float64, device="cuda")
        for c0 in range(0, nb, self.CHUNK):
            c = min(self.CHUNK, nb - c0)
            px, py, qx, qy, init = config5_host_inputs(slra, seed, self.b0 + c0, c)
            dev = [torch.from_numpy(a).cuda() for a in (px, py, qx, qy)]
            slra.gen_log_kernel_blocks_device(*[d.data_ptr() for d in dev], c, m, m, self.A[c0].data_ptr(), m, m * m)
            for i, d in enumerate(dev):
                self.pts[i, c0:c0 + c] = d.view(c, m)
            self.init[c0:c0 + c] = torch.from_numpy(init).cuda()
        torch.cuda.synchronize()
        self.I = torch.zeros(nb, C5_K, dtype=torch.int64, device="cuda")
        self.J = torch.zeros(nb, C5_K, dtype=torch.int64, device="cuda")
        self.U = torch.zeros(nb, C5_K * C5_K, dtype=torch.float64, device="cuda")
        self.r = torch.zeros(nb, dtype=torch.int64, device="cuda")
        self.st = torch.zeros(nb, dtype=torch.int32, device="cuda")
        self.rs = torch.zeros(nb, dtype=torch.float64, device="cuda")
        self.ns = torch.zeros(nb, dtype=torch.float64, device="cuda")
        self.entries_per_step = blocks * m * m  # the whole job (all ranks)
        self.data = ("synthetic (seeded; BASELINE config-5 recipe: per-block reference Rng; `value`: blocks "
                     "materialised in HBM; `e2e`: the blocks' points from pinned host memory, FunctionOracle)")
        self.config = config5_config(blocks)

    def step(self):
        self.slra.cross_approx_batched_device(self.A.data_ptr(), C5_M, C5_M * C5_M, self.nb, C5_M, C5_M, 0, C5_K,
                                              C5_K, self.init.data_ptr(), C5_LOOPS, 1.1, self.I.data_ptr(),
                                              self.J.data_ptr(), self.U.data_ptr(), self.r.data_ptr(),
                                              self.st.data_ptr(), self.rs.data_ptr(), self.ns.data_ptr())

    def last_residual_rel(self):
        rel = (self.rs / self.ns).sqrt()
        return {"max": float(rel.max().item()), "median": float(rel.median().item()),
                "failed_blocks": int((self.st != 0).sum().item()),
                "r_hist": {int(v): int(c) for v, c in zip(*torch_unique(self.torch, self.r))}}

    def cpu_baseline(self):
        """The oracle (reference path restated: cross_approx -> numerical_rank -> primitive_cur ->
        cur_evaluate) on a bounded sample of the same blocks (read back from HBM): ~10 s single-threaded
        (the reference runs one block per thread) and the same sample over all host cores."""
        sys.path.insert(0, os.path.join(ROOT, "oracle", "build"))
        import _oracle as oracle
        cores = os.cpu_count() or 1
        nall = min(self.nb, 8192)
        A_all = np.ascontiguousarray(self.A[:nall].cpu().numpy())
        init_all = self.init[:nall].cpu().numpy()
        A, init = A_all[:1024], init_all[:1024]
        # single thread: grow the sample until ~10 s
        n, dt1 = 16, 0.0
        while True:
            t0 = time.perf_counter()
            oracle_blocks(oracle, A[:n], init[:n], 1)
            dt1 = time.perf_counter() - t0
            if dt1 > 3.0 or n >= A.shape[0]:
                break
            n = min(A.shape[0], n * 4)
        t0 = time.perf_counter()
        oracle_blocks(oracle, A_all, init_all, cores)
        dtn = time.perf_counter() - t0
        return {"value": n * C5_M * C5_M / dt1, "unit": "entries/s", "cores": 1, "kind": "port",
                "sample": f"the first {n} config-5 blocks (read back from HBM) through the oracle/ C++ restatement "
                          f"of the reference path, one thread ({dt1:.1f} s); blocks are independent, so the rate "
                          f"extrapolates linearly",
                "all_cores": {"value": nall * C5_M * C5_M / dtn, "cores": cores,
                              "sample": f"the first {nall} blocks, one block per OpenMP thread ({dtn:.1f} s)"}}

    def roofline(self, fam, peaks, steps):
        kernels = {k: v[0] / steps for k, v in fam.items()}
        top = max(fam.items(), key=lambda kv: kv[1][0])[0]
        per = fam[top][0] / max(fam[top][1], 1)  # ms per launch
        flops = C5_FLOPS_PER_BLOCK * self.nb
        ach = flops / (per * 1e-3) / 1e12
        byts = C5_BYTES_PER_BLOCK * self.nb
        traffic = profiled_traffic(5, "ca_block_kernel", tag="r02", blocks=self.nb)
        return {"kernel": top + " (ca_block_kernel)", "bound": "tensor", "achieved": ach,
                "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                "frac": ach / peaks["fp64_tflops"] if peaks["fp64_tflops"] else None,
                "peak_source": peaks["fp64_source"],
                "algorithmic_per_launch": {"flops": flops, "bytes": byts,
                                           "basis": "SURVEY.md 8d config 5: 8.92 MFLOP and 512 KiB per block"},
                "traffic": traffic,
                "hbm_view": {"achieved_gbs": byts / (per * 1e-3) / 1e9,
                             "frac": byts / (per * 1e-3) / 1e9 / peaks["hbm_gbs"], "peak": peaks["hbm_gbs"]},
                "note": "FP64 latency-bound: one CTA per block (two per SM) runs the C-A chain (strip QR, "
                        "pivoted QR, maxvol, Jacobi SVD) and the DMMA residual; see DESIGN.md 5 and profiles/"}, kernels

    def function_oracle(self, steps, warmup):
        """The same batch with the blocks given by their points (FunctionOracle, oracle.hpp:43-54):
        slra_cross_approx_batched_logkernel evaluates every entry the C-A reads (strips, generator, the
        residual's full pass) from the points instead of reading a materialised block — bit-identical
        entries, so identical results (checked). Device-resident points (CUDA events), then the
        host-buffer entry (pinned points in, results out; wall clock)."""
        torch, slra, nb = self.torch, self.slra, self.nb
        outs = [torch.empty_like(t) for t in (self.I, self.J, self.U, self.r, self.st, self.rs, self.ns)]
        P = [self.pts[i].data_ptr() for i in range(4)]

        def dev():
            slra.cross_approx_batched_logkernel_device(*P, nb, C5_M, C5_M, 0, C5_K, C5_K, self.init.data_ptr(),
                                                       C5_LOOPS, 1.1, *[o.data_ptr() for o in outs])
        for _ in range(max(warmup, 1)):
            dev()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            dev()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        same = all(bool(torch.equal(a, b)) for a, b in zip(outs, (self.I, self.J, self.U, self.r, self.st, self.rs,
                                                                    self.ns)))
        return {"value": nb * C5_M * C5_M / (ms * 1e-3), "unit": "entries/s", "ms_per_step": ms, "steps": steps,
                "identical_to_dense_run": same,
                "api": "paper_1611_01391_b200.cross_approx_batched_logkernel_device -> "
                       "slra_cross_approx_batched_logkernel (device-resident points; blocks never materialised)"}

    def e2e(self, steps, warmup):
        """End to end with the blocks as the reference defines them for this config: an EntryOracle per
        block given by its points (FunctionOracle, oracle.hpp:43-54; K_ij = log|p_i - q_j|). Pinned host
        points in, every result (I, J, nucleus, r, status, residuals) back in pinned host memory, through
        slra_cross_approx_batched_logkernel_host; wall clock. The materialised-block variant of the same
        call is `e2e_dense_blocks` (host-link bound: 34 GB of blocks per step)."""
        torch, slra, nb = self.torch, self.slra, self.nb
        hp = [self.pts[i].cpu().pin_memory() for i in range(4)]
        hinit = self.init.cpu().pin_memory()
        houts = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True)
                 for o in (self.I, self.J, self.U, self.r, self.st, self.rs, self.ns)]

        def host():
            slra.cross_approx_batched_logkernel_host(*[h.data_ptr() for h in hp], nb, C5_M, C5_M, 0, C5_K, C5_K,
                                                     hinit.data_ptr(), C5_LOOPS, 1.1, *[o.data_ptr() for o in houts])
        for _ in range(max(1, min(warmup, 2))):
            host()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            host()
        dt = time.perf_counter() - t0
        same_host = all(bool(torch.equal(a, b.cpu())) for a, b in zip(houts, (self.I, self.J, self.U, self.r)))
        d2h = nb * (8 * 2 * C5_K + 8 * C5_K * C5_K + 8 + 4 + 16)
        return {"value": nb * C5_M * C5_M * steps / dt, "unit": "entries/s",
                "h2d_bytes_per_step": nb * 8 * (4 * C5_M + C5_K), "d2h_bytes_per_step": d2h,
                "steps": steps, "same_I_J_U_r_as_device_run": same_host,
                "input": "per-block points (FunctionOracle, oracle.hpp:43-54) + initial rows, pinned host memory",
                "api": "paper_1611_01391_b200.cross_approx_batched_logkernel_host -> "
                       "slra_cross_approx_batched_logkernel_host (points H2D, C-A + residual, results D2H)"}

    def e2e_dense(self, steps, warmup):
        """The batch through the host-buffer entry (slra_cross_approx_batched_host): pinned host blocks
        streamed to the device in chunks overlapped with the kernels, every result copied back."""
        torch = self.torch
        nb = self.nb
        host = torch.empty(nb * C5_M * C5_M, dtype=torch.float64, pin_memory=True)
        for c0 in range(0, nb, self.CHUNK):
            c = min(self.CHUNK, nb - c0)
            host[c0 * C5_M * C5_M:(c0 + c) * C5_M * C5_M].copy_(self.A[c0:c0 + c].reshape(-1))
        init = self.init.cpu().pin_memory()
        outs = [torch.empty(nb, C5_K, dtype=torch.int64, pin_memory=True),
                torch.empty(nb, C5_K, dtype=torch.int64, pin_memory=True),
                torch.empty(nb, C5_K * C5_K, dtype=torch.float64, pin_memory=True),
                torch.empty(nb, dtype=torch.int64, pin_memory=True),
                torch.empty(nb, dtype=torch.int32, pin_memory=True),
                torch.empty(nb, dtype=torch.float64, pin_memory=True),
                torch.empty(nb, dtype=torch.float64, pin_memory=True)]

        def one():
            self.slra.cross_approx_batched_host(host.data_ptr(), C5_M, C5_M * C5_M, nb, C5_M, C5_M, 0, C5_K, C5_K,
                                                init.data_ptr(), C5_LOOPS, 1.1, *[o.data_ptr() for o in outs])
        one()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        dt = time.perf_counter() - t0
        ok = bool(torch.equal(outs[0], self.I.cpu()) and torch.equal(outs[1], self.J.cpu()))
        d2h = nb * (8 * 2 * C5_K + 8 * C5_K * C5_K + 8 + 4 + 16)
        return {"value": self.nb * C5_M * C5_M * steps / dt, "unit": "entries/s",
                "h2d_bytes_per_step": nb * (8 * C5_M * C5_M + 8 * C5_K), "d2h_bytes_per_step": d2h,
                "steps": steps, "same_I_J_as_device_run": ok,
                "api": "paper_1611_01391_b200.cross_approx_batched_host -> slra_cross_approx_batched_host "
                       "(pinned host blocks in, chunked H2D overlapped with the C-A kernels; I, J, nucleus, r, "
                       "status, residuals out)"}


def torch_unique(torch, t):
    v, c = torch.unique(t, return_counts=True)
    return v.tolist(), c.tolist()


if __name__ == "__main__":
    main()
