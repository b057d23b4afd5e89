"""Compare the sharded scheduler (2 ranks on one GPU, gloo) with the single-
device engine after every step; prints the first divergence."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def wc(n, s):
    g = np.random.default_rng(s)
    m = g.uniform(-1, 1, (n, n))
    m[np.diag_indices(n)] += 2 * n
    return m


def worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    from paper_2305_11103_b200.distributed import ShardedEngine

    sizes = [64] * 8
    m = wc(512, 77)
    res = {}
    for s in range(1, 16):
        eng = ShardedEngine(sizes)
        eng.load(m)
        eng.run(1, s)
        res[s] = eng.gather()
    q.put((rank, res))
    dist.destroy_process_group()


if __name__ == "__main__":
    import paper_2305_11103_b200 as bi

    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get() for _ in range(2))
    for p in ps:
        p.join()
    m = wc(512, 77)
    for s in range(1, 16):
        single = bi.run_inversion(m, sizes=[64] * 8, stop_after_step=s).to_dense()
        d = np.abs(out[0][s] - single)
        print(s, "bitwise" if np.array_equal(out[0][s], single) else f"max diff {d.max():.3e} at {np.unravel_index(d.argmax(), d.shape)}")
