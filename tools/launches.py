"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel+grid."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
total = 0.0
for d in data:
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    k = d["Kernel Name"].split("(")[0][-40:] + " grid" + d["Grid Size"] + " blk" + d["Block Size"]
    agg[k][0] += 1
    agg[k][1] += v
    total += v
print(f"{len(data)} launches, {total:.1f} us total")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:5d} {t:11.1f} us {100 * t / total:5.1f}%  {t / c:9.2f} us/launch  {k}")
