"""Stall samples of one kernel grouped by execution count (loop body vs once-per-warp code),
from `ncu -i X --page source --csv --print-source sass`.  python tools/sass_regions.py sass.csv"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
reg, cnt = Counter(), Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    e = int(r[iE] or 0)
    reg[e] += int(r[iS] or 0)
    cnt[e] += 1
tot = sum(reg.values())
for e, s in sorted(reg.items(), key=lambda x: -x[1])[:8]:
    print(f"exec {e:6d}: {cnt[e]:5d} instructions, {s:6d} samples ({100 * s / tot:.1f} %)")
