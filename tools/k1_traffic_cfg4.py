"""DRAM traffic of the dominant kernel (K1) over one cfg4 engine run, from an
ncu CSV with dram__bytes_read.sum / dram__bytes_write.sum / gpu__time_duration.sum
per launch (tools/ncu_engine_range.py --cfg 4), against the algorithmic bytes
(bi_engine_counters out[5]: every operand read once, every output written
once).  Writes the JSON the bench's roofline.traffic reads.
    python tools/k1_traffic_cfg4.py launches.csv algorithmic_bytes out.json"""
import csv
import json
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = defaultdict(dict)
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if "gemm_tma_refill_kernel" not in d["Kernel Name"]:
        continue
    v = float(d["Metric Value"].replace(",", ""))
    per[d["ID"]][d["Metric Name"]] = v
n = len(per)
rd = sum(p.get("dram__bytes_read.sum", 0) for p in per.values())
wr = sum(p.get("dram__bytes_write.sum", 0) for p in per.values())
alg = float(sys.argv[2])
out = {"kernel": "gemm_tma_refill_kernel<4, 64>", "launches": n, "dram_bytes_read": rd, "dram_bytes_write": wr,
       "dram_bytes_per_launch": (rd + wr) / n, "algorithmic_bytes_per_launch": alg / n,
       "traffic_over_algorithmic": (rd + wr) / alg,
       "how": "ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
              "--clock-control none python tools/ncu_engine_range.py --cfg 4 (one cfg4 Eq. 7 run, every launch)"}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out))
