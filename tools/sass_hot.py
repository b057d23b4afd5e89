"""Per-instruction stall samples from `ncu -i X --page source --csv --print-source sass`.

  python tools/sass_hot.py sass.csv [min_samples]
Prints every instruction with >= min_samples samples, its top stall reasons,
and the total per stall reason."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 20
iS = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
tot = Counter()
total = 0
for k, r in enumerate(rows[2:]):
    if len(r) < len(hdr):
        continue
    s = int(r[iS] or 0)
    total += s
    st = {hdr[i][6:]: int(r[i] or 0) for i in stall_cols if r[i] not in ("", "0")}
    tot.update(st)
    if s >= lo:
        top = sorted(st.items(), key=lambda x: -x[1])[:3]
        print(f"{k:5d} {s:6d}  {r[1].strip()[:60]:60s} {top}")
print("total samples", total)
print(sorted(tot.items(), key=lambda x: -x[1])[:12])
