"""Checkpoint/resume format parity (storage.py:265-411,
core.py:421-484) on CPU: the product's writer reproduces a checkpoint
directory written by the REFERENCE byte for byte (fixture from
tests/golden/make_golden.py), its reader returns the reference state, and the
integrity checks raise the reference's errors."""

from pathlib import Path

import numpy as np
import pytest

import oracle
from conftest import well_conditioned
from tests_golden_inputs import GOLDEN

from paper_2305_11103_b200 import checkpoint as ckpt
from paper_2305_11103_b200.errors import CheckpointCorrupt, FormatError, SchemeMismatch

SIZES = [8] * 4
STOP = 4


def _golden_files():
    out = {}
    for k in GOLDEN.files:
        if k.startswith("ckpt4_file__"):
            out[k[len("ckpt4_file__"):].replace("__", "/")] = GOLDEN[k].tobytes()
    return out


def _oracle_state():
    m = well_conditioned(32, 61)
    minv, tsets = oracle.run_inversion(m, sizes=SIZES, stop_after_step=STOP, return_state=True)
    state = {}
    for level, t in tsets.items():
        entries = {}
        for kind in ("L", "R", "S"):
            for idx, arr in enumerate(t[kind]):
                if arr is not None:
                    entries[(kind, idx)] = arr
        if entries:
            state[level] = entries
    return m, minv, state


def test_bmat_roundtrip_and_errors(tmp_path):
    a = np.arange(6.0).reshape(2, 3) - 2.5
    ckpt.save_binary(a, tmp_path / "a.blk")
    assert (tmp_path / "a.blk").read_bytes()[:4] == b"BMAT"
    assert np.array_equal(ckpt.load_binary(tmp_path / "a.blk"), a)
    with pytest.raises(FormatError):
        ckpt.matrix_from_bytes(b"XMAT" + bytes(16))
    with pytest.raises(FormatError):
        ckpt.matrix_from_bytes(ckpt.matrix_to_bytes(a)[:-1])
    with pytest.raises(FormatError):
        ckpt.matrix_from_bytes(ckpt.matrix_to_bytes(np.array([[np.nan]])))


def test_writer_reproduces_reference_checkpoint_bytes(tmp_path):
    """oracle state after step 4 -> product writer == reference-written directory, every byte
    (incl. meta.json with the input fingerprint and the state hash)."""
    m, minv, state = _oracle_state()
    ckpt.checkpoint_save(tmp_path, SIZES, minv, state, STOP, ckpt.input_fingerprint(m, SIZES))
    golden = _golden_files()
    written = {str(p.relative_to(tmp_path)): p.read_bytes() for p in sorted(tmp_path.rglob("*")) if p.is_file()}
    assert sorted(written) == sorted(golden)
    for name, data in golden.items():
        assert written[name] == data, name


def test_reader_returns_reference_state_and_checks_integrity(tmp_path):
    for name, data in _golden_files().items():
        (tmp_path / name).parent.mkdir(parents=True, exist_ok=True)
        (tmp_path / name).write_bytes(data)
    meta = ckpt.checkpoint_load(tmp_path)
    m, minv_ref, state_ref = _oracle_state()
    assert meta["stepid"] == STOP and meta["sizes"] == SIZES and meta["blocksize"] == 4
    ckpt.checkpoint_matches(meta, SIZES, ckpt.input_fingerprint(m, SIZES))
    minv, state = ckpt.load_state(tmp_path, SIZES)
    assert minv.tobytes() == minv_ref.tobytes()
    assert {lv: sorted(e) for lv, e in state.items() if e} == {lv: sorted(e) for lv, e in state_ref.items()}
    for lv, entries in state_ref.items():
        for key, arr in entries.items():
            assert state[lv][key].tobytes() == arr.tobytes()
    other = m.copy()
    other[0, 0] += 1.0
    with pytest.raises(SchemeMismatch):
        ckpt.checkpoint_matches(meta, SIZES, ckpt.input_fingerprint(other, SIZES))
    with pytest.raises(SchemeMismatch):
        ckpt.checkpoint_matches(meta, [16, 16], ckpt.input_fingerprint(m, [16, 16]))
    victim = sorted(Path(tmp_path).rglob("*.blk"))[0]
    raw = bytearray(victim.read_bytes())
    raw[-1] ^= 0xFF
    victim.write_bytes(bytes(raw))
    with pytest.raises(CheckpointCorrupt):
        ckpt.checkpoint_load(tmp_path)


def test_missing_meta(tmp_path):
    with pytest.raises(CheckpointCorrupt):
        ckpt.checkpoint_load(tmp_path)  # test_storage.py:118-120


def _tree(root: Path) -> dict:
    return {str(p.relative_to(root)): p.read_bytes() for p in sorted(root.rglob("*")) if p.is_file()}


def test_incremental_writer_matches_checkpoint_save(tmp_path):
    """CheckpointWriter (the checkpointed run's writer: unchanged blocks are
    neither rewritten nor rehashed, the rest written on a thread pool) leaves
    the directory byte for byte as checkpoint_save does, step after step, and
    hashes files it did not write (a stale block) from disk like _state_hash."""
    sizes = [3, 5, 4, 4]
    n = sum(sizes)
    g = np.random.default_rng(9)
    minv = np.zeros((n, n))
    tsets: dict = {}
    ref_dir, new_dir = tmp_path / "ref", tmp_path / "new"
    new_dir.mkdir()
    (new_dir / "tset").mkdir()
    stale = np.arange(6.0).reshape(2, 3)
    for d in (ref_dir, new_dir):  # a block file neither writer produces
        (d / "tset").mkdir(parents=True, exist_ok=True)
        ckpt.save_binary(stale, d / "tset" / "stale.blk")
    writer = ckpt.CheckpointWriter(threads=3)
    for step in range(1, 6):
        i, j = g.integers(0, len(sizes), 2)  # this step touches one block of M_inv ...
        off = np.concatenate([[0], np.cumsum(sizes)])
        minv[off[i]:off[i + 1], off[j]:off[j + 1]] = g.standard_normal((sizes[i], sizes[j]))
        if step % 2 == 0:  # ... and every other step adds provisional entries
            tsets.setdefault(1, {})[("L", step)] = g.standard_normal((4, 3))
        ckpt.checkpoint_save(ref_dir, sizes, minv, tsets, step, "h")
        writer.save(new_dir, sizes, minv, tsets, step, "h")
        assert _tree(ref_dir) == _tree(new_dir), step
    assert ckpt.checkpoint_load(new_dir)["stepid"] == 5
