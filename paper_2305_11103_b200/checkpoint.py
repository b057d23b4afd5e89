"""Step-boundary checkpoint/resume of the device engine in the reference's
on-disk format, so a run can be staged across sessions and a
checkpoint written by either implementation can be resumed by the other.

Format (storage.py:265-411, core.py:421-484):
  <dir>/minv/B_<i>_<j>.blk        every block of M_inv (BMAT)
  <dir>/tset/<level>/<K>_<idx>.blk the provisional entries stored so far:
                                   L_q, R_q, S_{2q} (S_D), S_{2q+1} (S_A)
  <dir>/meta.json                  {version, stepid, blocksize, sizes,
                                    input_hash, state_hash}, written last
BMAT: b"BMAT", two little-endian u64 dims, float64 LE row-major.
state_hash = sha256("stepid=<s>\\n" + per sorted *.blk: relpath ":" sha256 "\\n").
input_hash = sha256(BMAT(m) + "|" + ",".join(sizes)).

The device engine keeps its state in HBM; a checkpoint is a D2H snapshot of
M_inv and of the T-set entries that exist after step s (every entry of level
l exists once the first arrows step at level l has run), written after every
step exactly like the reference's run_inversion (engine.py:527-539).
"""

from __future__ import annotations

import hashlib
import json
import os
import struct
from pathlib import Path

import numpy as np

from .errors import CheckpointCorrupt, DimensionMismatch, FormatError, SchemeMismatch

CHECKPOINT_VERSION = 1  # storage.py:36
_BMAT_MAGIC = b"BMAT"


# --- BMAT (core.py:421-484) -------------------------------------------------

def matrix_to_bytes(m) -> bytes:
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2:
        raise DimensionMismatch(f"expected a 2-D array, got ndim={m.ndim}")
    return _BMAT_MAGIC + struct.pack("<QQ", m.shape[0], m.shape[1]) + np.ascontiguousarray(m, dtype="<f8").tobytes()


def matrix_from_bytes(buf: bytes) -> np.ndarray:
    if len(buf) < 20 or buf[:4] != _BMAT_MAGIC:
        raise FormatError("missing BMAT magic")
    rows, cols = struct.unpack("<QQ", buf[4:20])
    if len(buf) != 20 + rows * cols * 8:
        raise FormatError(f"expected {20 + rows * cols * 8} bytes, got {len(buf)}")
    m = np.frombuffer(buf, dtype="<f8", offset=20).reshape(rows, cols)
    if m.shape[0] < 1 or m.shape[1] < 1:
        raise FormatError(f"bad matrix shape {m.shape}")
    if not np.all(np.isfinite(m)):
        raise FormatError("matrix contains NaN or Inf entries")
    return np.ascontiguousarray(m, dtype=np.float64)


def save_binary(m, path) -> None:
    Path(path).write_bytes(matrix_to_bytes(m))


def load_binary(path) -> np.ndarray:
    return matrix_from_bytes(Path(path).read_bytes())


# --- hashes and metadata (storage.py:270-360) --------------------------------

def input_fingerprint(m, sizes) -> str:
    h = hashlib.sha256()
    h.update(matrix_to_bytes(m))
    h.update(("|" + ",".join(map(str, sizes))).encode())
    return h.hexdigest()


def _blk_files(root: Path) -> list[Path]:
    return sorted(p for p in root.rglob("*.blk"))


def _state_hash(root: Path, stepid: int) -> str:
    h = hashlib.sha256()
    h.update(f"stepid={stepid}\n".encode())
    for path in _blk_files(root):
        h.update(str(path.relative_to(root)).encode())
        h.update(b":")
        h.update(hashlib.sha256(path.read_bytes()).hexdigest().encode())
        h.update(b"\n")
    return h.hexdigest()


def checkpoint_load(directory) -> dict:
    """meta.json after the integrity check (CheckpointCorrupt otherwise)."""
    root = Path(directory)
    meta_path = root / "meta.json"
    if not meta_path.exists():
        raise CheckpointCorrupt(f"no meta.json in {root}")
    try:
        meta = json.loads(meta_path.read_text())
    except (json.JSONDecodeError, OSError) as exc:
        raise CheckpointCorrupt(f"unreadable meta.json: {exc}") from exc
    for key in ("version", "stepid", "blocksize", "sizes", "input_hash", "state_hash"):
        if key not in meta:
            raise CheckpointCorrupt(f"meta.json missing {key!r}")
    if meta["version"] != CHECKPOINT_VERSION:
        raise CheckpointCorrupt(f"checkpoint version {meta['version']} unsupported")
    if _state_hash(root, meta["stepid"]) != meta["state_hash"]:
        raise CheckpointCorrupt("state hash mismatch")
    return meta


def checkpoint_matches(meta: dict, sizes, input_hash: str) -> None:
    if list(sizes) != list(meta["sizes"]) or len(sizes) != meta["blocksize"]:
        raise SchemeMismatch("partition scheme differs from checkpoint")
    if input_hash != meta["input_hash"]:
        raise SchemeMismatch("input matrix differs from checkpoint")


def has_checkpoint(directory) -> bool:
    return directory is not None and os.path.isdir(directory) and os.path.exists(os.path.join(directory, "meta.json"))


def clear_state(directory) -> None:
    """fresh_state for file-backed runs (storage.py:391-405): drop stale block
    files and meta.json so a new run cannot be confused with an old one."""
    root = Path(directory)
    if root.exists():
        for stale in _blk_files(root):
            os.remove(stale)
        meta = root / "meta.json"
        if meta.exists():
            meta.unlink()


# --- state <-> files ------------------------------------------------------------

def tset_entry_names(nb: int, level: int):
    """(kind, idx) in ProvisionalSet.entries() order (storage.py:257-262)."""
    nq = nb >> level
    return [("L", q) for q in range(nq)] + [("R", q) for q in range(nq)] + [("S", i) for i in range(2 * nq)]


def checkpoint_save(directory, sizes, minv: np.ndarray, tsets: dict, completed_step: int, input_hash: str) -> None:
    """Write the state after ``completed_step``: ``minv`` dense n x n,
    ``tsets`` {level: {(kind, idx): array}} (only entries that exist).
    meta.json last, so a torn save reads as corrupt rather than resumable."""
    root = Path(directory)
    root.mkdir(parents=True, exist_ok=True)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    mdir = root / "minv"
    mdir.mkdir(exist_ok=True)
    nb = len(sizes)
    for i in range(nb):
        for j in range(nb):
            save_binary(minv[off[i]:off[i + 1], off[j]:off[j + 1]], mdir / f"B_{i}_{j}.blk")
    for level, entries in tsets.items():
        tdir = root / "tset" / str(level)
        tdir.mkdir(parents=True, exist_ok=True)
        for (kind, idx), values in entries.items():
            save_binary(values, tdir / f"{kind}_{idx}.blk")
    meta = {
        "version": CHECKPOINT_VERSION,
        "stepid": completed_step,
        "blocksize": nb,
        "sizes": list(int(s) for s in sizes),
        "input_hash": input_hash,
        "state_hash": _state_hash(root, completed_step),
    }
    (root / "meta.json").write_text(json.dumps(meta, indent=1))


class CheckpointWriter:
    """checkpoint_save for the step loop of a checkpointed run: the same files
    and meta.json byte for byte, but a block whose values did not change since
    this writer's previous save is neither rewritten nor rehashed (each step
    touches only its own output blocks and new provisional entries), the
    remaining blocks are serialised, hashed and written on a thread pool
    (hashlib and file writes release the GIL), and the state hash comes from
    the hashes of the bytes just written instead of reading every file back.
    Files in the directory that this writer did not produce are hashed from
    disk, so the state hash is _state_hash's in every case."""

    def __init__(self, threads: int | None = None):
        self._cache: dict[str, tuple[str, np.ndarray]] = {}  # relpath -> (sha256 hex of the file, values)
        self._threads = threads or min(16, os.cpu_count() or 1)

    def save(self, directory, sizes, minv: np.ndarray, tsets: dict, completed_step: int, input_hash: str) -> None:
        from concurrent.futures import ThreadPoolExecutor

        root = Path(directory)
        root.mkdir(parents=True, exist_ok=True)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
        nb = len(sizes)
        blocks = []  # (relpath, array)
        (root / "minv").mkdir(exist_ok=True)
        for i in range(nb):
            for j in range(nb):
                blocks.append((f"minv/B_{i}_{j}.blk", minv[off[i]:off[i + 1], off[j]:off[j + 1]]))
        for level, entries in tsets.items():
            (root / "tset" / str(level)).mkdir(parents=True, exist_ok=True)
            for (kind, idx), values in entries.items():
                blocks.append((f"tset/{level}/{kind}_{idx}.blk", values))

        cache = self._cache

        def write(item):  # compare, and only if changed serialise, hash, write (numpy / hashlib / IO drop the GIL)
            rel, values = item
            hit = cache.get(rel)
            if hit is not None and hit[1].shape == values.shape and np.array_equal(hit[1], values) \
                    and (root / rel).exists():
                return None
            buf = matrix_to_bytes(values)
            (root / rel).write_bytes(buf)
            return rel, hashlib.sha256(buf).hexdigest(), np.array(values, dtype=np.float64, copy=True)

        with ThreadPoolExecutor(self._threads) as pool:
            for res in pool.map(write, blocks):
                if res is not None:
                    cache[res[0]] = (res[1], res[2])
        h = hashlib.sha256()
        h.update(f"stepid={completed_step}\n".encode())
        for path in _blk_files(root):
            rel = str(path.relative_to(root))
            hit = self._cache.get(rel)
            digest = hit[0] if hit is not None else hashlib.sha256(path.read_bytes()).hexdigest()
            h.update(rel.encode())
            h.update(b":")
            h.update(digest.encode())
            h.update(b"\n")
        meta = {
            "version": CHECKPOINT_VERSION,
            "stepid": completed_step,
            "blocksize": nb,
            "sizes": list(int(x) for x in sizes),
            "input_hash": input_hash,
            "state_hash": h.hexdigest(),
        }
        (root / "meta.json").write_text(json.dumps(meta, indent=1))


def load_state(directory, sizes):
    """(minv dense, {level: {(kind, idx): array}}) of a verified checkpoint."""
    root = Path(directory)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    nb = len(sizes)
    minv = np.zeros((off[-1], off[-1]))
    for i in range(nb):
        for j in range(nb):
            minv[off[i]:off[i + 1], off[j]:off[j + 1]] = load_binary(root / "minv" / f"B_{i}_{j}.blk")
    tsets = {}
    k = nb.bit_length() - 1
    for level in range(1, k + 1):
        tdir = root / "tset" / str(level)
        entries = {}
        if tdir.is_dir():
            for kind, idx in tset_entry_names(nb, level):
                p = tdir / f"{kind}_{idx}.blk"
                if p.exists():
                    entries[(kind, idx)] = load_binary(p)
        tsets[level] = entries
    return minv, tsets
