"""End-to-end time of the reference-signature Schur calls on NumPy arrays
(cfg3: n=6000, split 1000, singular A11 -> via_d), against the device-resident
formula.  Wall clock around the public call, warm, best of 5."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200 import _lib  # noqa: E402
from paper_2305_11103_b200.schur import schur2x2_device  # noqa: E402
from paper_2305_11103_b200.workloads import cfg3  # noqa: E402

m, split = cfg3()
n = m.shape[0]
out = np.empty_like(m)


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


md, od = _lib.to_device(m), _lib.empty_matrix(n, n)
t_dev = best(lambda: schur2x2_device("D", md, split, od))
t_fb = best(lambda: bi.invert_with_fallback(m, split, out))
q = bi.diagonal_quad(m, split)
t_d = best(lambda: bi.invert_via_d(q, bi.gpu_invert_sub, out))
res = bi.residual_frobenius(m, out)
print(f"cfg3 n={n}: device-resident via_d {t_dev:.1f} ms | invert_with_fallback(m, split, out) on NumPy {t_fb:.1f} ms "
      f"| invert_via_d(diagonal_quad(m), gpu_invert_sub, out) {t_d:.1f} ms | ||AX-I||_F {res:.2e}")
