"""Host-driven sharded schedule (distributed.py) at P = 1 vs the native graph
engine on cfg4 (n = 16384, 64 x 256): the per-GPU cost of the multi-GPU driver
before any communication."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200 import workloads  # noqa: E402
from paper_2305_11103_b200.distributed import run_inversion_local  # noqa: E402

m, sizes = workloads.cfg4()
for rep in range(2):
    t0 = time.perf_counter()
    out = run_inversion_local(m, sizes, 1)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
print(f"sharded driver P=1 (host-launched ops, incl. H2D/D2H of the full matrix): {1e3 * (t1 - t0):.1f} ms")
eng = bi.DeviceEngine(sizes, 1)
eng.load(m)
eng.run()
eng.check()
torch.cuda.synchronize()
t0 = time.perf_counter()
eng.run()
eng.check()
t1 = time.perf_counter()
print(f"native engine (graph, device-resident): {1e3 * (t1 - t0):.1f} ms")
ref = eng.Minv[0, :, :16384].cpu().numpy()
print("max |sharded - native| =", float(np.max(np.abs(out - ref))))
