"""CPU anchor for the reference arm (VERDICT r01 "next" #2).

Times the REAL reference package (``/root/reference/pkg/src``, imported in
this container only -- it cannot travel to the GPU box) on:

* one full cfg2 matrix (n=4096, 8 x 512, seed [2, 0]) at workers=1 and at
  workers=<every host thread>, with the reference's own timing protocol
  (bench.py:99-116: gc paused, ``release_mode()``), and
* the 64-block structure of cfg4 at reduced order (n=1024 64 x 16,
  n=2048 64 x 32), reference and oracle port side by side, so the port the
  bench's reference arm runs on the GPU box is pinned as a timing proxy and
  the n^3 extrapolation to n=16384 is anchored.

Writes one JSON object per measurement to stdout.
    python tools/cpu_anchor.py [--skip-cfg2]
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")


def timed(fn):
    from blockinv.core import release_mode

    gc_on = gc.isenabled()
    gc.disable()
    try:
        with release_mode():
            t0 = time.perf_counter()
            out = fn()
            return time.perf_counter() - t0, out
    finally:
        if gc_on:
            gc.enable()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-cfg2", action="store_true")
    args = ap.parse_args()
    import blockinv
    import oracle

    threads = len(os.sched_getaffinity(0))
    for n in (1024, 2048):
        g = np.random.default_rng(4)
        m = g.standard_normal((n, n)) / np.sqrt(n)
        m[np.diag_indices(n)] += 4.0
        sizes = [n // 64] * 64
        dt_ref, x = timed(lambda: blockinv.run_inversion(m, sizes=sizes, workers=1).to_dense())
        t0 = time.perf_counter()
        xo = oracle.run_inversion(m, sizes=sizes)
        dt_port = time.perf_counter() - t0
        print(json.dumps({"what": f"cfg4 structure n={n} 64x{n // 64}", "reference_s": dt_ref, "port_s": dt_port,
                          "reference_gflops_nominal": 2 * n ** 3 / dt_ref / 1e9,
                          "port_over_reference": dt_port / dt_ref,
                          "bitwise_equal": bool(np.array_equal(x, xo)),
                          "extrapolated_n16384_s": dt_ref * (16384 / n) ** 3}), flush=True)
    if args.skip_cfg2:
        return
    from paper_2305_11103_b200.workloads import cfg2

    ms, sizes = cfg2(1)
    m = ms[0]
    for w in (1, threads):
        dt, x = timed(lambda: blockinv.run_inversion(m, sizes=sizes, workers=w).to_dense())
        res = float(np.max(np.abs(m @ x - np.eye(m.shape[0]))))
        print(json.dumps({"what": "cfg2 matrix 0 (n=4096, 8 x 512)", "workers": w, "host_threads": threads,
                          "reference_s": dt, "reference_gflops_nominal": 2 * 4096 ** 3 / dt / 1e9,
                          "residual_max": res}), flush=True)


if __name__ == "__main__":
    main()
