"""Device time of the engine on cfg4 (Eq. 7 and pivot-A) and cfg2 (batch 4),
for A/B runs of library variants (BI_LIB=...):  python tools/ab_time.py"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200.workloads import cfg2, cfg4  # noqa: E402


def t(eng, reps):
    eng.run()
    eng.check()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        eng.run()
    b.record()
    torch.cuda.synchronize()
    eng.check()
    return a.elapsed_time(b) / reps


out = {"lib": os.environ.get("BI_LIB", "in-tree")}
m, sizes = cfg4()
for sched in (() if "--cfg2-only" in sys.argv else ("eq7", "pivot_a")):
    e = bi.DeviceEngine(sizes, schedule=sched)
    e.load(m)
    out[f"cfg4_{sched}_ms"] = t(e, 5)
    del e
    bi.release_engines()
ms, sizes = cfg2(4)
e = bi.DeviceEngine(sizes, batch=4)
e.load(ms)
out["cfg2_eq7_ms"] = t(e, 10)
print(json.dumps(out), flush=True)
