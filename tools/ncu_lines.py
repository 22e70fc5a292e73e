"""Attribute an ncu source-page (SASS) export to CUDA source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep OBJ.o KERNEL_MANGLED [top]

ncu's per-instruction samples / executed-instruction counts are joined with
`nvdisasm -g` line info of the same cubin (the object must be the one the
profiled library was linked from; compile with -lineinfo).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40

raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = None
ins = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        ins.append((int(d["Address"], 16), int(d["Warp Stall Sampling (All Samples)"] or 0),
                    int(d["Instructions Executed"] or 0), d["Source"].strip()))
base = ins[0][0]

with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    full = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cub)], capture_output=True, text=True).stdout
    start = full.index(f"//--------------------- .text.{fn} ")
    nxt = full.find("//--------------------- ", start + 10)
    sass = full[start:nxt if nxt > 0 else len(full)]
loc = {}
cur = ("?", 0)
for line in sass.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]+)\*/", line)
    if m:
        loc[int(m.group(1), 16)] = cur

agg = collections.defaultdict(lambda: [0, 0])
tot_s = tot_i = 0
for a, s, n, _ in ins:
    k = loc.get(a - base, ("?", 0))
    agg[k][0] += s
    agg[k][1] += n
    tot_s += s
    tot_i += n
print(f"samples {tot_s}  warp-instructions {tot_i}")
print(f"{'samp%':>6} {'inst%':>6}  file:line")
for k, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot_s:6.2f} {100 * n / tot_i:6.2f}  {k[0]}:{k[1]}")
