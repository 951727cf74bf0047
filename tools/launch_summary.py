"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: launches, total and mean duration, share of the listed time.
Usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) <= iv or not r[iv]:
        continue
    v = float(r[iv].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1.0)
    name = re.sub(r"\(.*", "", r[ik]).replace("void ", "")
    name = re.sub(r"<.*", "", name)
    agg[name].append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':34s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:34]:34s} {len(v):8d} {sum(v):10.1f} {sum(v) / len(v):9.2f} {100 * sum(v) / tot:5.1f}%")
