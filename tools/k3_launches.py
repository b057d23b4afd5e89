"""Launch list of ONE K3 call (device_inverse) for ncu:
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/k3_launches.py COUNT N
The call is warmed up first; only the second call is inside the profiler range."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_11103_b200 import _lib  # noqa: E402
from paper_2305_11103_b200.core import device_inverse  # noqa: E402

count, n = int(sys.argv[1]), int(sys.argv[2])
g = np.random.default_rng(3)
x = _lib.to_device(g.standard_normal((count, n, n)) + n * np.eye(n))
o = _lib.empty_matrix(n, n, batch=count)
device_inverse(x, o)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
device_inverse(x, o)
b.record()
torch.cuda.synchronize()
print(f"K3 {count} x {n}: {a.elapsed_time(b):.3f} ms (unprofiled)")
torch.cuda.profiler.start()
device_inverse(x, o)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
