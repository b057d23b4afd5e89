"""K3 device time for batches of equal blocks (graph-free, CUDA events, warm):
    python tools/k3_time.py 64x256 8x512 32x512"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402
from paper_2305_11103_b200 import _lib  # noqa: E402
from paper_2305_11103_b200.core import device_inverse  # noqa: E402

for spec in sys.argv[1:]:
    cnt, n = (int(x) for x in spec.split("x"))
    g = np.random.default_rng(11)
    x = g.standard_normal((cnt, n, n)) + n * np.eye(n)
    dx = _lib.to_device(x)
    do = _lib.empty_matrix(n, n, batch=cnt)
    for _ in range(3):
        device_inverse(dx, do, sync=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        device_inverse(dx, do, sync=False)
    b.record()
    torch.cuda.synchronize()
    err = max(oracle.rel_frob(do[i].cpu().numpy(), np.linalg.inv(x[i])) for i in range(min(cnt, 4)))
    print(f"K3 {spec}: {a.elapsed_time(b) / reps:.3f} ms  relF {err:.1e}", flush=True)
