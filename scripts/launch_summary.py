"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel.

    python scripts/launch_summary.py gpurun_out/launches.csv [steps]
"""
import collections
import csv
import sys

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = list(csv.reader(open(path)))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        us = v / 1000 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1000)
        k = d["Kernel Name"][:100]
        agg[k][0] += 1
        agg[k][1] += us
tot = sum(v[1] for v in agg.values()) / steps
print(f"total {tot / 1000:.2f} ms per step ({steps} steps in list)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{v[1] / steps / 1000:7.3f} ms {v[0] // steps:5d}x {v[1] / v[0]:8.2f} us  {k}")
