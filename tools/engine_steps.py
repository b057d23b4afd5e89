"""Per-step cost model inputs for the lane scheduler (cfg2 shape): GEMM flops
per step (bi_engine_counters), and the per-step timeline of ONE lane running
alone (batch 1) -- what each step costs when nothing overlaps it.

  python tools/engine_steps.py
"""
import os
import sys
from pathlib import Path

os.environ["BI_ENGINE_TIMELINE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200 import _lib  # noqa: E402
from paper_2305_11103_b200.workloads import cfg2  # noqa: E402

ms, sizes = cfg2(1)
eng = bi.DeviceEngine(sizes, batch=1)
eng.load(ms)
for _ in range(3):
    eng.run()
eng.check()
ns = eng.n_steps
buf = (_lib.ctypes.c_float * (ns + 1))()
_lib.check(_lib.lib().bi_engine_timeline(eng._h, buf), "bi_engine_timeline")
t = np.array(buf[:], dtype=np.float64)
print("step gemm_GF leaf_GF alone_ms")
prev = 0.0
for st in range(1, ns + 1):
    c = eng.counters(st, st)
    print(f"{st:4d} {c['gemm_flops'] / 1e9:8.2f} {c['leaf_flops'] / 1e9:7.2f} {t[st] - prev:8.3f}")
    prev = t[st]
print("total alone", t[ns])
