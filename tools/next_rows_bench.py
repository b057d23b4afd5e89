"""Measurement of the SURVEY 8(f) rows beside the hot path (one B200; CUDA
events / wall clock, warm; each result checked):

  * the single-level formulas of schur.py on the device (bi_schur2x2): the
    diagonal pivots A (Eq. 2), D (Eq. 3), AD (Eq. 7) and the counter-diagonal
    pivots B, C, BC (8f #2) at n = 6000 with a 3000 split, residual-checked;
  * checkpointed run_inversion (8f #3): one cfg2-structure matrix (n = 4096,
    8 x 512) with a checkpoint after every step in the reference's on-disk
    format, against the plain run, and a resume from the step-7 checkpoint;
  * the reference CLI on the device (8f #4): `invert` of the same matrix from
    a binary file, process wall time.

    python tools/next_rows_bench.py
"""
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200 import _lib  # noqa: E402
from paper_2305_11103_b200.schur import schur2x2_device  # noqa: E402
from paper_2305_11103_b200.workloads import cfg2  # noqa: E402


def ev_time(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def formulas():
    n, p = 6000, 3000
    g = np.random.default_rng(61)
    m = g.standard_normal((n, n)) / np.sqrt(n) + 4.0 * np.eye(n)
    # the counter-diagonal pivots need invertible B / C: put the dominant part there too
    mc = g.standard_normal((n, n)) / np.sqrt(n)
    mc[:p, p:] += 4.0 * np.eye(p)
    mc[p:, :p] += 4.0 * np.eye(p)
    for pivot, mat, label in (("A", m, "via_a (Eq. 2)"), ("D", m, "via_d (Eq. 3)"), ("X", m, "via_ad (Eq. 7)"),
                              ("B", mc, "via_b"), ("C", mc, "via_c"), ("Y", mc, "via_bc")):
        md = _lib.to_device(mat)
        out = _lib.empty_matrix(n, n)
        ms = ev_time(lambda: schur2x2_device(pivot, md, p, out))
        res = bi.residual_frobenius(mat, out.cpu().numpy())
        print(f"{label:16s} n={n} split={p}: {ms:8.2f} ms = {2 * n ** 3 / ms / 1e9:6.2f} TF/s nominal  "
              f"||AX-I||_F {res:.2e}", flush=True)


def checkpointing():
    ms, sizes = cfg2(1)
    m = ms[0]
    n = m.shape[0]
    plain = ev_time(lambda: bi.run_inversion(m, sizes=sizes), reps=3)
    ref = bi.run_inversion(m, sizes=sizes).to_dense()
    with tempfile.TemporaryDirectory() as d:
        t0 = time.perf_counter()
        got = bi.run_inversion(m, sizes=sizes, checkpoint_dir=d).to_dense()
        t_ck = time.perf_counter() - t0
        size = sum(f.stat().st_size for f in Path(d).rglob("*") if f.is_file())
        assert np.array_equal(got, ref)
    with tempfile.TemporaryDirectory() as d:
        bi.run_inversion(m, sizes=sizes, checkpoint_dir=d, stop_after_step=7)
        t0 = time.perf_counter()
        got = bi.run_inversion(m, sizes=sizes, checkpoint_dir=d).to_dense()
        t_res = time.perf_counter() - t0
        assert np.array_equal(got, ref)
    print(f"run_inversion n={n} (8 x 512, 15 steps): plain {plain:.1f} ms; checkpoint after every step "
          f"{t_ck * 1e3:.0f} ms ({size / 2**20:.0f} MiB on disk at the end); resume from step 7 -> 15 "
          f"{t_res * 1e3:.0f} ms; both bitwise equal to the plain run", flush=True)


def cli():
    ms, sizes = cfg2(1)
    m = ms[0]
    with tempfile.TemporaryDirectory() as d:
        src, dst = os.path.join(d, "m.bin"), os.path.join(d, "inv.bin")
        bi.save_binary(m, src)
        cmd = [sys.executable, "-m", "paper_2305_11103_b200", "invert", "--in", src, "--out", dst, "--binary",
               "--method", "parallel", "--sizes", ",".join(str(s) for s in sizes)]
        walls = []
        for _ in range(3):
            t0 = time.perf_counter()
            r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
            walls.append(time.perf_counter() - t0)
            assert r.returncode == 0, r.stderr[-2000:]
        inv = bi.load_binary(dst)
        res = bi.residual_frobenius(m, inv)
        print(f"CLI invert n={m.shape[0]} (binary file in/out, --method parallel): process wall "
              f"{min(walls):.2f} s (best of 3, incl. interpreter + torch import + library load)  "
              f"||AX-I||_F {res:.2e}", flush=True)


if __name__ == "__main__":
    formulas()
    checkpointing()
    cli()
