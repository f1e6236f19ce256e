"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name (ms, launches).
  python tools/launch_summary.py LAUNCHES.csv [top]"""
import collections
import csv
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for r in csv.DictReader(lines):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0][:90]
    agg[name][0] += 1
    agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
tot = sum(a[1] for a in agg.values())
print(f"launches {sum(a[0] for a in agg.values())}  total {tot:.2f} ms")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{t:10.2f} ms {c:5d}  {k}")
