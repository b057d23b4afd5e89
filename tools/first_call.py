"""First-call latency of run_inversion in a fresh process (engine bind, tensor
maps, CUDA-graph capture) against the warm call, cfg2 one matrix and cfg4."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
t_imp = time.perf_counter()
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200.workloads import cfg2, cfg4  # noqa: E402

torch.cuda.init()
print(f"import {time.perf_counter() - t_imp:.2f} s", flush=True)
for name, (m, sizes) in (("cfg2 one matrix", (cfg2(1)[0][0], cfg2(1)[1])), ("cfg4", cfg4())):
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bi.run_inversion(m, sizes=sizes)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    print(f"{name}: first call {times[0] * 1e3:.0f} ms, then {times[1] * 1e3:.0f} / {times[2] * 1e3:.0f} ms", flush=True)
