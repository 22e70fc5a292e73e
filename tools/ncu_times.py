"""Summarise an ncu --csv gpu__time_duration log: per kernel name, count and mean/total us."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0][:60] + " " + d["Grid Size"]
        v = float(d["Metric Value"]) / 1000.0
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
for k, (n, t) in agg.items():
    print(f"{n:5d} {t / n:10.2f} us  {t:10.2f} us  {k}")
