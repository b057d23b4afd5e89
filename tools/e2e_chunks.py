"""cfg4 end to end through run_inversion(m) on a NumPy array vs device time
(BI_OUT_CHUNKS A/B helper).  CUDA events, warm, 3 reps."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200.workloads import cfg4  # noqa: E402

m, sizes = cfg4()


def timed(fn, reps=3):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


print(f"run_inversion(m) {timed(lambda: bi.run_inversion(m, sizes=sizes)):.2f} ms", flush=True)
