"""The reference algorithm (oracle port, bitwise equal to the reference) on
ONE full cfg2 matrix on the GPU box's host cores, at one process and with
every host thread busy (one matrix per process: the batch of 4 and more),
anchoring the bench's n^3 extrapolation.  ~5 min.
    python tools/cpu_anchor_box.py"""
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def one(b: int) -> float:
    import oracle
    from paper_2305_11103_b200.workloads import cfg2

    rng = np.random.default_rng([2, b % 4])
    m = rng.standard_normal((4096, 4096)) / 64.0
    m[np.diag_indices(4096)] += 2.0
    t0 = time.perf_counter()
    oracle.run_inversion(m, sizes=[512] * 8)
    return time.perf_counter() - t0


if __name__ == "__main__":
    threads = len(os.sched_getaffinity(0))
    t1 = one(0)
    print(json.dumps({"what": "cfg2 matrix 0, oracle port, 1 process", "s": t1,
                      "gflops_nominal": 2 * 4096 ** 3 / t1 / 1e9}), flush=True)
    with mp.get_context("fork").Pool(threads) as pool:
        t0 = time.perf_counter()
        ts = pool.map(one, range(threads), chunksize=1)
        wall = time.perf_counter() - t0
    print(json.dumps({"what": f"cfg2 matrices, oracle port, {threads} processes (one matrix each)", "wall_s": wall,
                      "per_matrix_s": ts, "aggregate_gflops_nominal": threads * 2 * 4096 ** 3 / wall / 1e9}),
          flush=True)
