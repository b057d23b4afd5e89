"""End-to-end latency of the reference-signature API (NumPy in, NumPy out):
run_inversion(m, sizes=...) on one cfg2 matrix and on cfg4, as a user calls it
(host copies included, engine cached after the first call)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200 import workloads  # noqa: E402


def lat(fn, reps):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    return (time.perf_counter() - t0) / reps, out


ms, sizes = workloads.cfg2(1)
m2 = ms[0]
t, inv = lat(lambda: bi.run_inversion(m2, sizes=sizes).to_dense(), 5)
print(f"cfg2 one matrix (n=4096, 8x512): run_inversion {1e3 * t:.1f} ms  "
      f"({2 * 4096**3 / t / 1e12:.1f} TF/s nominal), residual_F {bi.residual_frobenius(m2, inv):.2e}")
t, inv = lat(lambda: bi.run_inversion(m2, sizes=sizes, schedule='pivot_a').to_dense(), 5)
print(f"cfg2 one matrix, schedule='pivot_a': {1e3 * t:.1f} ms")
m4, sizes4 = workloads.cfg4()
t, inv = lat(lambda: bi.run_inversion(m4, sizes=sizes4).to_dense(), 2)
print(f"cfg4 (n=16384, 64x256): run_inversion {1e3 * t:.1f} ms ({2 * 16384**3 / t / 1e12:.1f} TF/s nominal)")
t, inv = lat(lambda: bi.run_inversion(m4, sizes=sizes4, schedule='pivot_a').to_dense(), 2)
print(f"cfg4, schedule='pivot_a': {1e3 * t:.1f} ms ({2 * 16384**3 / t / 1e12:.1f} TF/s nominal)")
