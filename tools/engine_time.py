"""Device time of the step engine on cfg4 (one 16384 matrix, 64 x 256) and the
cfg2 batch (4 x 4096, 8 x 512), Eq. 7 schedule, CUDA events, warm:
    python tools/engine_time.py [cfg4] [cfg2] [--reps R]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200.workloads import cfg2, cfg4  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("which", nargs="*", default=["cfg4", "cfg2"])
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
for w in args.which:
    if w == "cfg4":
        m, sizes = cfg4()
        ms = m[None]
    else:
        ms, sizes = cfg2(4)
    eng = bi.DeviceEngine(sizes, batch=ms.shape[0])
    eng.load(ms)
    for _ in range(2):
        eng.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        eng.run()
    e1.record()
    torch.cuda.synchronize()
    print(f"{w}: {e0.elapsed_time(e1) / args.reps:.2f} ms per run", flush=True)
