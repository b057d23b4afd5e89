"""Device checkpoint/resume: run_inversion(checkpoint_dir=...,
file_backed=...) with the reference's semantics (test_storage.py:66-140): a
resumed run is bitwise equal to an uninterrupted device run; a checkpoint
written by the REFERENCE resumes on the device; integrity and scheme checks."""

from pathlib import Path

import numpy as np
import pytest

import oracle
from conftest import well_conditioned
from tests_golden_inputs import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bi():
    import paper_2305_11103_b200 as bi

    return bi


def test_resume_bitwise_after_partial_run(bi, tmp_path):
    m = well_conditioned(21, 52)
    ref = bi.run_inversion(m).to_dense()
    for stop in (1, 7, 14):
        d = tmp_path / f"ck{stop}"
        bi.run_inversion(m, checkpoint_dir=d, stop_after_step=stop)
        out = bi.run_inversion(m, checkpoint_dir=d).to_dense()
        assert out.tobytes() == ref.tobytes(), stop


def test_file_backed_resume_bitwise_and_completed(bi, tmp_path):
    m = well_conditioned(64, 53)
    sizes = [8] * 8
    ref = bi.run_inversion(m, sizes=sizes).to_dense()
    d = tmp_path / "ck"
    bi.run_inversion(m, sizes=sizes, checkpoint_dir=d, file_backed=True, stop_after_step=8)
    out = bi.run_inversion(m, sizes=sizes, checkpoint_dir=d, file_backed=True).to_dense()
    assert out.tobytes() == ref.tobytes()
    again = bi.run_inversion(m, sizes=sizes, checkpoint_dir=d).to_dense()  # completed checkpoint
    assert again.tobytes() == ref.tobytes()
    with pytest.raises(ValueError):
        bi.run_inversion(m, sizes=sizes, file_backed=True)


def test_checkpoint_errors(bi, tmp_path):
    m = well_conditioned(12, 55)
    d = tmp_path / "ck"
    bi.run_inversion(m, checkpoint_dir=d, stop_after_step=2)
    other = m.copy()
    other[0, 0] += 1.0
    with pytest.raises(bi.SchemeMismatch):
        bi.run_inversion(other, checkpoint_dir=d)
    with pytest.raises(bi.SchemeMismatch):
        bi.run_inversion(m, checkpoint_dir=d, sizes=[6, 6])
    victim = sorted(Path(d).rglob("*.blk"))[0]
    raw = bytearray(victim.read_bytes())
    raw[-1] ^= 0xFF
    victim.write_bytes(bytes(raw))
    with pytest.raises(bi.CheckpointCorrupt):
        bi.run_inversion(m, checkpoint_dir=d)


def test_device_state_matches_oracle_state(bi, tmp_path):
    """The state the device writes after step s is the reference engine's state
    after step s (oracle, GJ leaves) to 1e-12, entry by entry."""
    from paper_2305_11103_b200 import checkpoint as ckpt

    sizes = [8] * 8
    m = well_conditioned(64, 45)
    for stop in (3, 8, 12):
        d = tmp_path / f"s{stop}"
        bi.run_inversion(m, sizes=sizes, checkpoint_dir=d, stop_after_step=stop)
        assert ckpt.checkpoint_load(d)["stepid"] == stop
        minv, state = ckpt.load_state(d, sizes)
        ref_minv, ref_t = oracle.run_inversion(m, sizes=sizes, stop_after_step=stop, return_state=True,
                                               leaf_inverter=oracle.gauss_jordan)
        assert np.max(np.abs(minv - ref_minv)) <= 1e-12 * max(1.0, np.max(np.abs(ref_minv)))
        for lv, t in ref_t.items():
            for kind in ("L", "R", "S"):
                for idx, arr in enumerate(t[kind]):
                    if arr is None:
                        assert (kind, idx) not in state.get(lv, {})
                    else:
                        got = state[lv][(kind, idx)]
                        assert np.max(np.abs(got - arr)) <= 1e-12 * max(1.0, np.max(np.abs(arr))), (lv, kind, idx)


def test_reference_written_checkpoint_resumes_on_device(bi, tmp_path):
    """Directory written by the reference after step 4 of 7 (golden bytes) ->
    device resume -> the reference's full-run inverse to 1e-12."""
    for k in GOLDEN.files:
        if k.startswith("ckpt4_file__"):
            p = tmp_path / k[len("ckpt4_file__"):].replace("__", "/")
            p.parent.mkdir(parents=True, exist_ok=True)
            p.write_bytes(GOLDEN[k].tobytes())
    m = well_conditioned(32, 61)
    out = bi.run_inversion(m, sizes=[8] * 4, checkpoint_dir=tmp_path).to_dense()
    assert oracle.rel_frob(out, GOLDEN["ckpt4_final"]) <= 1e-12
    assert bi.checkpoint_load(tmp_path)["stepid"] == 7
