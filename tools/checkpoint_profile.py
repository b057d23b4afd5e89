"""Per-phase time of the checkpointed step loop (run / snapshot / save), cfg2-structure matrix."""
import sys, time, tempfile
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2305_11103_b200 as bi
from paper_2305_11103_b200 import checkpoint as ckpt
from paper_2305_11103_b200.engine import _engine_for
from paper_2305_11103_b200.workloads import cfg2
ms, sizes = cfg2(1); m = ms[0]
eng = _engine_for(tuple(sizes), 1); eng.load(m)
w = ckpt.CheckpointWriter()
tr = ts = tw = 0.0
with tempfile.TemporaryDirectory() as d:
    for s in range(1, 16):
        t0 = time.perf_counter(); eng.run(s, s, use_graph=False); eng.check(); t1 = time.perf_counter()
        minv, tsets = eng.snapshot(s); t2 = time.perf_counter()
        w.save(d, sizes, minv, tsets, s, "h"); t3 = time.perf_counter()
        tr += t1 - t0; ts += t2 - t1; tw += t3 - t2
print(f"run {tr*1e3:.0f} ms, snapshot {ts*1e3:.0f} ms, save {tw*1e3:.0f} ms over 15 steps")
