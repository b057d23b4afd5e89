"""Host-buffer entry points of the engine (bi_engine_run_host) against the
device-resident run, bitwise:

* pageable NumPy input: the engine's need-ordered staging (level by level,
  chunked DMA under the compute, run_host_pipelined) -- with page-locked and
  with pageable output (staged read-back), batch 1 and batch > 1, both
  schedules, stop_after_step states, ragged partitions, inputs whose row
  pitch exceeds n (views into a wider array);
* page-locked input (graph-captured copies, round 1);
* the public run_inversion / run_inversion_batch on plain NumPy arrays,
  including repeated calls that reuse the cached staging and page-locked
  results, and SingularBlock reporting through the pageable path.
"""

import numpy as np
import pytest
import torch

import oracle
from conftest import well_conditioned

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bi():
    import paper_2305_11103_b200 as bi

    return bi


def _device_ref(bi, ms, sizes, schedule="eq7", last=None):
    eng = bi.DeviceEngine(sizes, batch=ms.shape[0], schedule=schedule)
    eng.load(ms)
    eng.run(1, last)
    eng.check()
    n = ms.shape[1]
    return eng.Minv[:, :, :n].cpu().numpy()


def _batch(sizes, batch, seed):
    n = sum(sizes)
    return np.stack([well_conditioned(n, seed + b) for b in range(batch)])


@pytest.mark.parametrize("sizes,batch", [([64] * 8, 1), ([64] * 8, 3), ([37, 29, 51, 16, 44, 23, 60, 8], 2),
                                         ([128] * 16, 1), ([300, 212], 1)])
@pytest.mark.parametrize("out_kind", ["pinned", "pageable"])
def test_pageable_input_bitwise(bi, sizes, batch, out_kind):
    ms = _batch(sizes, batch, 40 + batch)
    ref = _device_ref(bi, ms, sizes)
    eng = bi.DeviceEngine(sizes, batch=batch)
    out = (torch.empty(ms.shape, dtype=torch.float64, pin_memory=True).numpy() if out_kind == "pinned"
           else np.empty_like(ms))
    for _ in range(2):  # the second call reuses the staging and the cached range graphs
        out[...] = np.nan
        eng.run_host(ms, out)
        eng.check()
        assert np.array_equal(out, ref)


@pytest.mark.parametrize("stop", [1, 2, 3, 6, 9, 15])
def test_pageable_stop_after_step(bi, stop):
    sizes = [48] * 8
    ms = _batch(sizes, 1, 7)
    ref = _device_ref(bi, ms, sizes, last=stop)
    got = bi.run_inversion(ms[0], sizes=sizes, stop_after_step=stop).to_dense()
    assert np.array_equal(got, ref[0])


def test_pageable_pivot_a(bi):
    sizes = [96] * 8
    ms = _batch(sizes, 2, 3)
    ref = _device_ref(bi, ms, sizes, schedule="pivot_a")
    got = bi.run_inversion_batch(ms, sizes, schedule="pivot_a")
    assert np.array_equal(got, ref)


def test_input_view_with_wider_rows(bi):
    """Row pitch > n: a view into a wider array goes through the staging."""
    sizes = [40] * 8
    n = sum(sizes)
    wide = np.zeros((n, n + 17))
    wide[:, 5:5 + n] = well_conditioned(n, 21)
    view = wide[:, 5:5 + n]
    assert not view.flags.c_contiguous
    eng = bi.DeviceEngine(sizes)
    out = np.empty((n, n))
    eng.run_host(view, out)
    eng.check()
    assert np.array_equal(out, _device_ref(bi, np.ascontiguousarray(view)[None], sizes)[0])


def test_pinned_input_matches_pageable(bi):
    sizes = [64] * 8
    ms = _batch(sizes, 2, 11)
    eng = bi.DeviceEngine(sizes, batch=2)
    pin = torch.from_numpy(ms).pin_memory().numpy()
    a = torch.empty(ms.shape, dtype=torch.float64, pin_memory=True).numpy()
    b = np.empty_like(ms)
    eng.run_host(pin, a)
    eng.check()
    eng.run_host(ms, b)
    eng.check()
    assert np.array_equal(a, b)


def test_public_api_repeated_and_oracle(bi):
    sizes = [32, 96, 64, 64]
    n = sum(sizes)
    m = well_conditioned(n, 5)
    first = bi.run_inversion(m, sizes=sizes).to_dense()
    for _ in range(3):
        assert np.array_equal(bi.run_inversion(m, sizes=sizes).to_dense(), first)
    ref = oracle.run_inversion(m, sizes=sizes, leaf_inverter=oracle.gauss_jordan)
    assert oracle.rel_frob(first, ref) <= 1e-12


def test_pageable_singular_reported(bi):
    sizes = [32] * 8
    n = sum(sizes)
    m = well_conditioned(n, 9)
    m[96:128, 96:128] = 0.0  # diagonal block 3 singular at step 1
    with pytest.raises(bi.SingularBlock) as ei:
        bi.run_inversion(m, sizes=sizes)
    assert (ei.value.step, ei.value.quad) == (1, 3)
    # the engine stays usable afterwards
    good = well_conditioned(n, 10)
    assert oracle.residual_max(good, bi.run_inversion(good, sizes=sizes).to_dense()) <= 1e-8 * n


def test_pageable_batch_more_lanes_than_streams(bi):
    """batch 10 > 8 lanes: lanes carry two matrices; need-ordered staging
    over every matrix of every level."""
    sizes = [24] * 8
    ms = _batch(sizes, 10, 70)
    ref = _device_ref(bi, ms, sizes)
    got = bi.run_inversion_batch(ms, sizes)
    assert np.array_equal(got, ref)


_RING_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2305_11103_b200 as bi
from conftest import well_conditioned
for sizes, batch in (([64] * 8, 1), ([37, 29, 51, 16, 44, 23, 60, 8], 3), ([128] * 16, 2)):
    n = sum(sizes)
    ms = np.stack([well_conditioned(n, 90 + b) for b in range(batch)])
    eng = bi.DeviceEngine(sizes, batch=batch)
    eng.load(ms); eng.run(); eng.check()
    ref = eng.Minv[:, :, :n].cpu().numpy()
    out = np.full_like(ms, np.nan)
    eng.run_host(ms, out); eng.check()
    assert np.array_equal(out, ref), sizes
    for stop in (1, 4):
        e2 = bi.DeviceEngine(sizes, batch=batch); e2.load(ms); e2.run(1, stop); e2.check()
        o2 = np.full_like(ms, np.nan); eng.run_host(ms, o2, 1, stop); eng.check()
        assert np.array_equal(o2, e2.Minv[:, :, :n].cpu().numpy()), (sizes, stop)
print("ring ok")
"""


def test_ring_path_for_buffers_above_the_staging_limit(tmp_path):
    """Host buffers above BI_STAGE_LIMIT_GB go through the bounded page-locked
    ring (run_host_ring): forced here with a tiny limit and 64 KB slots so
    pieces split across slots and every slot is reused many times."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, BI_STAGE_LIMIT_GB="1e-6", BI_RING_MB="0.0625",
               PYTHONPATH=os.pathsep.join([str(root), str(root / "tests")]))
    script = tmp_path / "ring.py"
    script.write_text(_RING_SCRIPT)
    r = subprocess.run([sys.executable, str(script), str(root)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ring ok" in r.stdout, r.stdout + r.stderr


_CHUNKS_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2305_11103_b200 as bi
from conftest import well_conditioned
for sizes, batch in (([64] * 8, 1), ([37, 29, 51, 16, 44, 23, 60, 8], 2), ([128] * 16, 1)):
    n = sum(sizes)
    ms = np.stack([well_conditioned(n, 120 + b) for b in range(batch)])
    eng = bi.DeviceEngine(sizes, batch=batch)
    eng.load(ms); eng.run(); eng.check()
    ref = eng.Minv[:, :, :n].cpu().numpy()
    pin_in = torch.from_numpy(ms).pin_memory().numpy()
    pin_out = torch.full(ms.shape, float("nan"), dtype=torch.float64, pin_memory=True).numpy()
    eng.run_host(pin_in, pin_out); eng.check()
    assert np.array_equal(pin_out, ref), sizes
print("chunks ok")
"""


@pytest.mark.parametrize("chunks", ["1", "3", "16"])
def test_last_pass_read_back_chunks(tmp_path, chunks):
    """The last top-level pass runs in BI_OUT_CHUNKS row chunks, each read back
    as soon as it is written (page-locked output): any chunk count gives the
    device-resident inverse bitwise, ragged partitions and batches included."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, BI_OUT_CHUNKS=chunks, PYTHONPATH=os.pathsep.join([str(root), str(root / "tests")]))
    script = tmp_path / "chunks.py"
    script.write_text(_CHUNKS_SCRIPT)
    r = subprocess.run([sys.executable, str(script), str(root)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "chunks ok" in r.stdout, r.stdout + r.stderr
