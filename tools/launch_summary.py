"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("msg::", "")
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':28s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:28s} {v[0]:8d} {v[1]:10.1f} {v[1] / v[0]:8.2f} {100 * v[1] / tot:5.1f}%")
print(f"total kernel time {tot / 1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches")
