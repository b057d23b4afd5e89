"""Host-driven sharded schedule (P = 1, cfg4): wall vs device time and a cProfile."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_11103_b200 import workloads  # noqa: E402
from paper_2305_11103_b200.distributed import ShardedEngine  # noqa: E402
from paper_2305_11103_b200.local_group import LocalWorld  # noqa: E402

m, sizes = workloads.cfg4()
eng = ShardedEngine(sizes, dist=LocalWorld(1).facade(0))
eng.load(m)
eng.run()
eng.check()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
eng.run()
e1.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
eng.check()
print(f"enqueue (host) {1e3 * (t1 - t0):.1f} ms, wall to completion {1e3 * (t2 - t0):.1f} ms, "
      f"device {e0.elapsed_time(e1):.1f} ms")
pr = cProfile.Profile()
pr.enable()
eng.run()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
