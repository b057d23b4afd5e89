"""GPU: the opt-in tuning knobs (DESIGN 8) keep results correct.  Each knob is
read once per process, so every combination runs in a fresh interpreter
(six interpreters at a time):
K3 alone (n = 300 / 512 / 1000) and the engine (8 x 64 and 4 x 128 blocks)
against the oracle, relF <= 1e-12 / 1e-9."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
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
    {"BI_GJ_FUSED": "1"},
    {"BI_GJ_FUSED": "1", "BI_GJ_FAST": "0"},
    {"BI_GJ_FAST_SMALL": "1"},
    {"BI_GEMM_WARPS": "4"},
    {"BI_GEMM_WARPS": "8"},
    {"BI_GEMM_TM": "64"},
    {"BI_ENGINE_PDL": "1"},
    {"BI_GJ_SUBLA": "1"},
    {"BI_GJ_SUBLA": "1", "BI_GJ_FAST_SMALL": "1"},
]


def _knob_id(k: dict) -> str:
    return ",".join(f"{a}={b}" for a, b in k.items())


@pytest.fixture(scope="module")
def knob_runs():
    """Every combination's interpreter, six at a time (most of a run is the
    interpreter start and the CPU oracle, not the GPU): the per-knob tests
    below only collect their own result."""
    from concurrent.futures import ThreadPoolExecutor

    def run(knobs):
        env = dict(os.environ, **knobs)
        return subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, capture_output=True, text=True,
                              timeout=600)

    pool = ThreadPoolExecutor(max_workers=6)
    futures = {_knob_id(k): pool.submit(run, k) for k in KNOBS}
    yield futures
    pool.shutdown(wait=False, cancel_futures=True)


@pytest.mark.parametrize("knobs", KNOBS, ids=_knob_id)
def test_knob_combination_correct(knobs, knob_runs):
    r = knob_runs[_knob_id(knobs)].result(timeout=1200)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]


BITWISE_GEMM = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
from paper_2305_11103_b200 import _lib
L = _lib.lib()
g = torch.Generator(device="cuda").manual_seed(5)
outs = []
for m, n, k, batch, acc in ((1024, 1024, 1024, 2, True), (640, 200, 1100, 3, False), (2048, 512, 4096, 1, True),
                            (300, 300, 300, 2, True)):
    a = torch.randn(batch, m, k, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(batch, k, n, dtype=torch.float64, device="cuda", generator=g)
    c = torch.randn(batch, m, n, dtype=torch.float64, device="cuda", generator=g) if acc else None
    d = torch.empty(batch, m, n, dtype=torch.float64, device="cuda")
    rc = L.bi_gemm(m, n, k, 1, a.data_ptr(), k, m * k, b.data_ptr(), n, k * n,
                   c.data_ptr() if acc else None, n if acc else 0, m * n if acc else 0,
                   d.data_ptr(), n, m * n, batch, _lib.stream_ptr())
    assert rc == 0
    outs.append(d.cpu().numpy())
np.savez(sys.argv[2], *outs)
print("ok")
"""


@pytest.mark.parametrize("variant", [{"BI_GEMM_WARPS": "4"}, {"BI_GEMM_TM": "64"}], ids=["warps4", "tm64"])
def test_gemm_tile_variants_bitwise(tmp_path, variant):
    """K1's tile variants -- 4 warps of 64 x 32, 64 x 64 CTA tiles -- sum every
    element in the same order as the 8-warp 128 x 64 tile: bitwise equal
    outputs, including ragged shapes."""
    res = {}
    base = {"BI_GEMM_WARPS": "8", "BI_GEMM_TM": "128"}
    for w, knobs in (("v", variant), ("base", base)):
        f = tmp_path / f"{w}.npz"
        env = dict(os.environ, **knobs)
        r = subprocess.run([sys.executable, "-c", BITWISE_GEMM, str(ROOT), str(f)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        res[w] = np.load(f)
    for key in res["v"].files:
        assert np.array_equal(res["v"][key], res["base"][key]), key


@pytest.mark.parametrize("knob", ["BI_GJ_FUSED", "BI_GJ_SUBLA"])
def test_k3_variants_bitwise(knob):
    """BI_GJ_FUSED=1 (one cluster launch per batch of blocks <= 512) and
    BI_GJ_SUBLA=1 (sub-panel lookahead) are bitwise the multi-launch chain, on
    dominant, random, permuted, singular, ragged and tied blocks
    (tools/k3_fast_check.py)."""
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "k3_fast_check.py"), knob], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "ALL BITWISE EQUAL" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
