"""A K3 knob at 1 against 0, bitwise: BI_GJ_FAST=1 (verified diagonal-pivot
panels) against the pivoted column loop, or BI_GJ_FUSED=1 (the fused
single-launch cluster kernel for n <= 512) against the multi-launch chain.
Inverses and info must be bitwise equal on diagonally dominant blocks (fast
path taken), random blocks (fallback), singular and permuted blocks,
batches, ragged orders and a large cluster-panel block.
    python tools/k3_fast_check.py [KNOB]     # driver: runs both modes, compares
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
CASES = [("dom", 64, 256), ("dom", 8, 512), ("rand", 8, 256), ("rand", 4, 512), ("perm", 4, 256),
         ("sing", 4, 256), ("dom", 1, 5000), ("rand", 1, 3000), ("dom", 3, 100), ("mixed", 16, 200),
         ("dom", 1, 1000), ("tie", 2, 64), ("dom", 2, 300), ("perm", 2, 512), ("dom", 3, 129), ("rand", 3, 24),
         ("sing", 2, 512), ("rand", 2, 384)]


def make(kind, cnt, n, seed):
    g = np.random.default_rng(seed)
    if kind == "dom":
        x = g.standard_normal((cnt, n, n)) / np.sqrt(n) + 4 * np.eye(n)
    elif kind == "rand":
        x = g.standard_normal((cnt, n, n))
    elif kind == "perm":
        x = np.stack([np.eye(n)[g.permutation(n)] + 1e-3 * g.standard_normal((n, n)) for _ in range(cnt)])
    elif kind == "sing":
        x = g.standard_normal((cnt, n, n)) / np.sqrt(n) + 4 * np.eye(n)
        x[:, 40:48, :] = 0.0
    elif kind == "tie":
        x = np.stack([np.eye(n) * 2.0 + np.diag(np.full(n - 1, 2.0), -1) for _ in range(cnt)])
    else:
        x = g.standard_normal((cnt, n, n)) / np.sqrt(n) + 4 * np.eye(n)
        x[::2] = g.standard_normal((cnt - cnt // 2, n, n))
    return x


def child(out_dir):
    sys.path.insert(0, str(ROOT))
    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.core import device_inverse

    for ci, (kind, cnt, n) in enumerate(CASES):
        x = make(kind, cnt, n, 100 + ci)
        do = _lib.empty_matrix(n, n, batch=cnt)
        info = device_inverse(_lib.to_device(x), do, sync=False)
        info = np.asarray(info.cpu() if hasattr(info, "cpu") else info)
        np.save(os.path.join(out_dir, f"c{ci}_x.npy"), do.cpu().numpy())
        np.save(os.path.join(out_dir, f"c{ci}_i.npy"), info)


if __name__ == "__main__":
    if len(sys.argv) > 1 and not sys.argv[1].startswith("BI_"):
        child(sys.argv[1])
        sys.exit(0)
    import tempfile

    knob = sys.argv[1] if len(sys.argv) > 1 else "BI_GJ_FAST"
    on = "1"
    if "=" in knob:  # KNOB=VALUE: compare VALUE against 0
        knob, on = knob.split("=", 1)
    print(f"{knob}=0 vs {knob}={on}")
    outs = {}
    for mode in ("0", on):
        d = tempfile.mkdtemp()
        env = dict(os.environ, **{knob: mode})
        subprocess.run([sys.executable, __file__, d], env=env, check=True)
        outs[mode] = d
    ok = True
    for ci, (kind, cnt, n) in enumerate(CASES):
        a = np.load(os.path.join(outs["0"], f"c{ci}_x.npy"))
        b = np.load(os.path.join(outs[on], f"c{ci}_x.npy"))
        ia = np.load(os.path.join(outs["0"], f"c{ci}_i.npy"))
        ib = np.load(os.path.join(outs[on], f"c{ci}_i.npy"))
        same = np.array_equal(a, b, equal_nan=True) and np.array_equal(ia, ib)
        ok &= same
        print(f"{kind:5s} {cnt:3d} x {n:5d}: bitwise {'equal' if same else 'DIFFERENT'}  info {ia.tolist()[:4]}")
    print("ALL BITWISE EQUAL" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)
