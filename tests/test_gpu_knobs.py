"""GPU: the opt-in tuning knobs (DESIGN 8) keep results correct.  Each knob is
read once per process, so every combination runs in a fresh interpreter:
K3 alone (n = 300 / 512 / 1000) and the engine (8 x 64 and 4 x 128 blocks)
against the oracle, relF <= 1e-12 / 1e-9."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
import oracle
import paper_2305_11103_b200 as bi
from paper_2305_11103_b200 import _lib
from paper_2305_11103_b200.core import device_inverse
from conftest import well_conditioned

for n, count in ((300, 3), (512, 4), (1000, 1)):
    ms = np.stack([well_conditioned(n, 50 + n + i) for i in range(count)])
    out = _lib.empty_matrix(n, n, batch=count)
    info = device_inverse(_lib.to_device(ms), out)
    assert not info.any(), (n, info)
    got = out.cpu().numpy()
    for i in range(count):
        err = oracle.rel_frob(got[i], oracle.gauss_jordan(ms[i]))
        assert err <= 1e-12, (n, i, err)
for sizes in ([64] * 8, [128] * 4):
    m = well_conditioned(sum(sizes), 77)
    inv = bi.run_inversion(m, sizes=sizes).to_dense()
    assert oracle.rel_frob(inv, oracle.gauss_jordan(m)) <= 1e-9
print("ok")
"""

KNOBS = [
    {"BI_GJ_LOOKAHEAD": "1"},
    {"BI_GJ_NB": "16"},
    {"BI_PDL": "0"},
    {"BI_GJ_CLUSTER": "2"},
    {"BI_GEMM_TMA": "0", "BI_GEMM_CP_TN": "128"},
    {"BI_GEMM_TN": "128", "BI_GEMM_REFILL": "0"},
    {"BI_PRIORITY_MODE": "4", "BI_ENGINE_SKEW": "1", "BI_RESERVE_SMS": "16"},
]


@pytest.mark.parametrize("knobs", KNOBS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()))
def test_knob_combination_correct(knobs):
    env = dict(os.environ, **knobs)
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
