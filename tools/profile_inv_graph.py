"""K3 batched inversion (count x n) timed host-launched and replayed from a
CUDA graph: the difference is the inter-kernel launch overhead."""
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
ap.add_argument("--count", type=int, default=8)
args = ap.parse_args()
g = np.random.default_rng(0)
ms = g.standard_normal((args.count, args.n, args.n)) / np.sqrt(args.n) + 2 * np.eye(args.n)
dm = _lib.to_device(ms)
out = _lib.empty_matrix(args.n, args.n, batch=args.count)
for _ in range(3):
    device_inverse(dm, out)
torch.cuda.synchronize()


def timed(fn, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


L = _lib.lib()
ws = _lib.workspace(L.bi_inv_workspace_bytes(args.count, args.n))
info = torch.zeros(args.count, dtype=torch.int32, device="cuda")


def raw():
    rc = L.bi_inv_batched(args.count, args.n, _lib.ptr(dm), _lib.ld(dm), int(dm.stride(0)), _lib.ptr(out),
                          _lib.ld(out), int(out.stride(0)), _lib.ctypes.c_void_p(info.data_ptr()), _lib.ptr(ws),
                          ws.numel(), _lib.stream_ptr())
    assert rc == 0


raw()
torch.cuda.synchronize()
t_host = timed(raw)
s = torch.cuda.Stream()
graph = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    raw()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=s):
        raw()
torch.cuda.synchronize()
t_graph = timed(graph.replay)
print(f"inv {args.count}x{args.n}: host-launched {t_host:.3f} ms, graph replay {t_graph:.3f} ms")
