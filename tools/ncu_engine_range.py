"""One engine run (or a step range) of a config inside a cudaProfilerStart/Stop
range, warmed up first, for ncu --profile-from-start off:

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \\
      python tools/ncu_engine_range.py --cfg 4                 # launch list of one cfg4 run
  ncu --profile-from-start off --set full --clock-control none \\
      python tools/ncu_engine_range.py --cfg 4 --steps 64 64   # the level-6 arrows step (2 K1 launches)
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200.workloads import cfg2, cfg4  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4, choices=(2, 4))
ap.add_argument("--steps", type=int, nargs=2, default=None)
args = ap.parse_args()
if args.cfg == 4:
    m, sizes = cfg4()
    ms = m[None]
else:
    ms, sizes = cfg2(4)
eng = bi.DeviceEngine(sizes, batch=ms.shape[0])
eng.load(ms)
eng.run()
eng.check()
first, last = args.steps if args.steps else (1, eng.n_steps)
if first > 1:
    eng.run(1, first - 1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.run(first, last, use_graph=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
eng.check()
print("counters", eng.counters(first, last))
