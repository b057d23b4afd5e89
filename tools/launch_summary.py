"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per kernel
name, launches and total/mean time."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    ns = v * {"ns": 1, "nsecond": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
    k = d["Kernel Name"][:90]
    agg[k][0] += 1
    agg[k][1] += ns
tot = sum(v[1] for v in agg.values())
print(f"total {tot / 1e3:.1f} us over {sum(v[0] for v in agg.values())} launches")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t / 1e3:10.1f} us {c:5d} x {t / c / 1e3:8.2f} us  {100 * t / tot:5.1f}%  {k}")
