"""Drop-in conformance: the reference's OWN test suite run against this
framework, and the reference's own Schur formulas calling the B200 leaf
through their plugin protocol.

  python tools/reference_suite.py --prepare   # here: copy the reference tests and package
                                              # into baseline/_ref/ (git-ignored; travels to the box)
  python tools/reference_suite.py --run       # on the GPU box: writes gpurun_out/reference_suite.txt

--run:
 1. pytest on baseline/_ref/tests with ``blockinv`` resolved to this package
    (tools/refshim): every test of the reference, unmodified; the summary
    lists each failure next to its documented divergence.
 2. The REAL reference package (baseline/_ref/src) -- its invert_via_d and
    invert_with_fallback (schur.py:142-164, 300-333) -- with
    paper_2305_11103_b200.gpu_invert_sub as ``invert_sub``.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/pkg")
DEST = ROOT / "baseline" / "_ref"

PLUGIN_DEMO = r'''
import sys, json, numpy as np
import blockinv
from blockinv.schur import diagonal_quad, invert_via_d, invert_with_fallback
from blockinv.core import gauss_jordan_oracle
import paper_2305_11103_b200 as bi
from paper_2305_11103_b200.workloads import cfg3
assert "reference" in blockinv.__file__ or "_ref" in blockinv.__file__, blockinv.__file__
out = {}
for n, split, rank in ((900, 150, 75), (6000, 1000, 500)):
    m, split = cfg3(n=n, split=split, rank=rank)
    x = np.empty_like(m)
    invert_via_d(diagonal_quad(m, split), bi.gpu_invert_sub, x)       # reference formula, B200 leaf
    res = float(np.linalg.norm(m @ x - np.eye(n)))
    y = np.empty_like(m)
    name = invert_with_fallback(m, split, y, invert_sub=bi.gpu_invert_sub)  # reference fallback order
    ref = np.linalg.inv(m)
    out[f"n={n}"] = {"via_d_residual_fro": res, "bound_n_eps_cond": n * np.finfo(float).eps * np.linalg.cond(m),
                     "via_d_relF_vs_lapack": float(np.linalg.norm(x - ref) / np.linalg.norm(ref)),
                     "fallback_returned": name, "fallback_equals_via_d": bool(np.array_equal(x, y))}
print(json.dumps(out, indent=1))
'''


def prepare() -> None:
    DEST.mkdir(parents=True, exist_ok=True)
    for sub, src in (("tests", REF / "tests"), ("src/blockinv", REF / "src" / "blockinv")):
        dst = DEST / sub
        if dst.exists():
            shutil.rmtree(dst)
        shutil.copytree(src, dst, ignore=shutil.ignore_patterns("__pycache__"))
    print(f"copied the reference tests and package into {DEST} (git-ignored)")


def run() -> None:
    outdir = ROOT / "gpurun_out"
    outdir.mkdir(exist_ok=True)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tools" / "refshim"), str(ROOT)])
    cmd = [sys.executable, "-m", "pytest", str(DEST / "tests"), "-q", "-rfE", "-p", "no:cacheprovider",
           "--continue-on-collection-errors",
           "--rootdir", str(DEST / "tests"), "-o", "addopts="]
    r = subprocess.run(cmd, cwd=str(DEST / "tests"), env=env, capture_output=True, text=True)
    env2 = dict(os.environ)
    env2["PYTHONPATH"] = os.pathsep.join([str(DEST / "src"), str(ROOT)])
    d = subprocess.run([sys.executable, "-c", PLUGIN_DEMO], cwd=str(ROOT), env=env2, capture_output=True, text=True)
    with open(outdir / "reference_suite.txt", "w") as f:
        f.write("# 1. reference test suite (baseline/_ref/tests = /root/reference/pkg/tests, unmodified),\n"
                "#    blockinv -> paper_2305_11103_b200 (tools/refshim), on one B200\n")
        f.write(r.stdout[-20000:])
        f.write(r.stderr[-4000:])
        f.write(f"\n# pytest rc={r.returncode}\n\n# 2. the real reference's invert_via_d / invert_with_fallback "
                "with invert_sub=paper_2305_11103_b200.gpu_invert_sub\n")
        f.write(d.stdout)
        f.write(d.stderr[-4000:])
        f.write(f"# demo rc={d.returncode}\n")
    print((outdir / "reference_suite.txt").read_text()[-6000:])


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--prepare", action="store_true")
    ap.add_argument("--run", action="store_true")
    a = ap.parse_args()
    if a.prepare:
        prepare()
    if a.run:
        run()
