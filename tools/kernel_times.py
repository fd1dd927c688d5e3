"""Per-kernel device time (ncu launch list) summary: python tools/kernel_times.py launches.csv"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}
    us = v * scale.get(unit, 1.0)
    agg[name].append(us)
for k, v in agg.items():
    print(f"{k[:70]:70s} n={len(v):3d} mean={sum(v)/len(v):9.2f} us  min={min(v):9.2f}")
