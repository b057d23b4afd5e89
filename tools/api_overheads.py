"""Wall time of reference-signature calls on NumPy arrays (best of 5, warm),
next to the size of the data they move: where host-side overhead remains."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402


def best(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


g = np.random.default_rng(5)
for n in (512, 2048, 4096):
    x0 = g.standard_normal((n, n)) / np.sqrt(n) + 4 * np.eye(n)
    x = x0.copy()

    def inplace():
        x[...] = x0
        bi.invertor_inplace_by_a(x)

    t_ip = best(inplace)
    t_ba = best(lambda: bi.invertor_by_a(x0))
    out = np.empty_like(x0)
    t_sub = best(lambda: bi.gpu_invert_sub(x0, out))
    a, b, c = (g.standard_normal((n, n)) for _ in range(3))
    t_mul = best(lambda: bi.multiply(a, b, c))
    t_ri = best(lambda: bi.run_inversion(x0, sizes=[n // 8] * 8))
    print(f"n={n:5d} ({x0.nbytes / 2**20:6.1f} MiB): invertor_inplace_by_a {t_ip:7.2f} ms | invertor_by_a {t_ba:7.2f} | "
          f"gpu_invert_sub {t_sub:7.2f} | multiply {t_mul:7.2f} | run_inversion 8 blocks {t_ri:7.2f}", flush=True)
