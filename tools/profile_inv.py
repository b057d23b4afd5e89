"""Drive one batched K3 inversion (count x n) for ncu / timing."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_11103_b200 import _lib  # noqa: E402
from paper_2305_11103_b200.core import device_inverse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--count", type=int, default=32)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--fast", action="store_true", help="pointer-table form (bi_inv_batched_ptrs)")
args = ap.parse_args()
g = np.random.default_rng(0)
ms = g.standard_normal((args.count, args.n, args.n)) / np.sqrt(args.n) + 2 * np.eye(args.n)
dm = _lib.to_device(ms)
out = _lib.empty_matrix(args.n, args.n, batch=args.count)
if args.fast:
    from paper_2305_11103_b200.core import device_inverse_list

    blocks, outs = [dm[i] for i in range(args.count)], [out[i] for i in range(args.count)]
    run = lambda: device_inverse_list(blocks, outs).cpu().numpy()  # noqa: E731
else:
    run = lambda: device_inverse(dm, out)  # noqa: E731
for _ in range(args.reps):
    info = run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
ms_ = e0.elapsed_time(e1)
print(f"inv {args.count}x{args.n}: {ms_:.3f} ms, {args.count * 2 * args.n**3 / ms_ / 1e9:.2f} TF/s, info max {info.max()}")
