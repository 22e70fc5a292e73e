"""Summarise the ncu outputs of tools/profile_round.sh into profiles/.

usage: python tools/summarize_profiles.py TAG CONFIG
writes profiles/TAG_cCONFIG_launches.txt (per-kernel launch times),
       profiles/TAG_cCONFIG_ncu_full.md (key counters per captured kernel),
       profiles/TAG_cCONFIG_traffic.json (DRAM bytes per launch, read by bench.py).
"""
import collections
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG, CFG = sys.argv[1], sys.argv[2]
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

# 1. launch list
rows = list(csv.reader(open(os.path.join(OUT, f"{TAG}_c{CFG}_launches.csv"))))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0] + " grid=" + d["Grid Size"]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"]) / 1000.0
tot = sum(t for _, t in agg.values())
with open(os.path.join(PROF, f"{TAG}_c{CFG}_launches.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n")
    f.write(f"# bench.py --config {CFG} --steps 2 --warmup 3: all launches of our kernels in the process\n")
    f.write(f"{'launches':>8} {'mean_us':>10} {'total_us':>11} {'share':>6}  kernel\n")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{n:8d} {t / n:10.2f} {t:11.2f} {100 * t / tot:5.1f}%  {k}\n")

# 2. full captures
WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "instructions"),
]
traffic = {}
lines = [f"# ncu --set full captures, {TAG}, bench.py --config {CFG}\n",
         "One launch per kernel (`-c 1`, first launch after start-up), --clock-control none.\n"]
for rep in sorted(glob.glob(os.path.join(OUT, f"{TAG}_c{CFG}_full_*.ncu-rep"))):
    name = os.path.basename(rep)[len(f"{TAG}_c{CFG}_full_"):-len(".ncu-rep")]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) < 3:
        continue
    d = dict(zip(rr[0], rr[2]))
    u = dict(zip(rr[0], rr[1]))
    lines.append(f"\n## {name}\n\n| counter | value |\n|---|---|\n")
    for key, label in WANT:
        if key in d:
            lines.append(f"| {label} (`{key}`) | {d[key]} {u.get(key, '')} |\n")
    stalls = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v))
              for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")]
    stalls = sorted([s for s in stalls if s[1] > 0.05], key=lambda s: -s[1])[:6]
    lines.append("| top stall reasons (warps per issue) | " + ", ".join(f"{k} {v:.2f}" for k, v in stalls) + " |\n")

    def num(key):
        v = d.get(key, "0").replace(",", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(key, "byte"), 1)
        return float(v) * scale
    dur = float(d.get("gpu__time_duration.sum", "0").replace(",", ""))
    dur_ms = dur * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}.get(
        u.get("gpu__time_duration.sum", "ms"), 1.0)
    traffic[name] = {"dram_bytes": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
                     "duration_ms": dur_ms, "grid": d.get("launch__grid_size", "")}
with open(os.path.join(PROF, f"{TAG}_c{CFG}_ncu_full.md"), "w") as f:
    f.writelines(lines)
with open(os.path.join(PROF, f"{TAG}_c{CFG}_traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1)
print(open(os.path.join(PROF, f"{TAG}_c{CFG}_launches.txt")).read())
print(json.dumps(traffic, indent=1))
