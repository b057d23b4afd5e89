"""Step-scheduled inversion of a matrix partitioned into 2**k diagonal blocks,
on the B200.

Mirrors /root/reference/pkg/src/blockinv/engine.py: the same stepid -> loopid
-> action schedule (engine.py:73-162) and the same public entry points, with
the step interpreter replaced by the native scheduler in libblockinv_b200.so
(``bi_engine_*``).  All state -- M, M_inv and every provisional set T_l --
stays resident in HBM for the whole run; a run is one CUDA-graph replay.

Extension (allowed by SURVEY 8d for config 2): ``run_inversion_batch`` inverts
a batch of matrices that share one partition in lock-step, so every leaf /
GEMM launch covers the whole batch.
"""

from __future__ import annotations

import os
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import OpCounters
from .errors import (
    BlockShapeMismatch,
    DimensionMismatch,
    MalformedLoopid,
    OutOfRange,
    SchemeMismatch,
    SingularBlock,
)
from .partition import PartitionScheme, make_partition, partition_from_sizes
from .storage import BlockMatrix, MemoryBlockStore

INVERT_DIAGONALS = "invert_diagonals"
ARROWS_AND_SCHUR = "arrows_and_schur"
SCHUR_DIAG_AND_ASSEMBLE = "schur_diag_and_assemble"


def resolve_workers(explicit: int | None = None) -> int:
    """Explicit argument beats INVERTOR_WORKERS (engine.py:58-65).  On the
    B200 build it is the GPU count for run_inversion (gpus_for_workers): the
    schedule is column-sharded over that many GPUs of this process; the
    result does not depend on it (K is never split)."""
    if explicit is not None:
        if explicit < 1:
            raise ValueError(f"workers must be >= 1, got {explicit}")
        return explicit
    env = os.environ.get("INVERTOR_WORKERS", "").strip()
    return max(int(env), 1) if env else 1


# ---------------------------------------------------------------------------
# schedule (host integer logic; the native scheduler decodes identically)
# ---------------------------------------------------------------------------


def total_steps(blocksize: int) -> int:
    """engine.py:73-74."""
    return 2 * blocksize - 1


def loopid_for_step(stepid: int, blocksize: int) -> list[int]:
    """Descending 1-based set-bit positions of stepid, zero-padded to
    log2(blocksize)+1 entries (engine.py:77-90)."""
    if blocksize < 1 or blocksize & (blocksize - 1):
        raise OutOfRange(f"blocksize must be a power of two, got {blocksize}")
    if not 1 <= stepid <= total_steps(blocksize):
        raise OutOfRange(f"stepid {stepid} outside 1..{total_steps(blocksize)}")
    width = blocksize.bit_length()
    bits = [b + 1 for b in range(width - 1, -1, -1) if (stepid >> b) & 1]
    return bits + [0] * (width - len(bits))


@dataclass(frozen=True)
class StepAction:
    """Decoded meaning of one step (engine.py:93-107)."""

    kind: str
    source: str
    cid: int | None = None
    sid: int | None = None
    depth: int = 0


@dataclass(frozen=True)
class StepPlan:
    stepid: int
    loopid: tuple
    action: StepAction


def decode_step(loopid) -> StepAction:
    """The loopid rules of engine.py:117-157."""
    loopid = list(loopid)
    nz: list[int] = []
    zero_seen = False
    for v in loopid:
        if v == 0:
            zero_seen = True
        elif zero_seen or v < 0:
            raise MalformedLoopid(f"{loopid}: zeros only as suffix")
        else:
            nz.append(v)
    if not nz:
        raise MalformedLoopid(f"{loopid}: no nonzero elements")
    if any(x <= y for x, y in zip(nz, nz[1:])):
        raise MalformedLoopid(f"{loopid}: prefix not strictly decreasing")
    last = nz[-1]
    if len(nz) == 1:
        if last == 1:
            return StepAction(INVERT_DIAGONALS, "matrix")
        return StepAction(ARROWS_AND_SCHUR, "matrix", sid=last - 1)
    cid = nz[-2] - 1
    if last == 1:
        run = 1
        while run < len(nz) and nz[-run - 1] == run + 1:
            run += 1
        return StepAction(SCHUR_DIAG_AND_ASSEMBLE, "tset", cid=cid, depth=run - 1)
    return StepAction(ARROWS_AND_SCHUR, "tset", cid=cid, sid=last - 1)


def step_plan(stepid: int, blocksize: int) -> StepPlan:
    loopid = loopid_for_step(stepid, blocksize)
    return StepPlan(stepid, tuple(loopid), decode_step(loopid))


def updown_iteration_map(block_row: int, block_col: int) -> int:
    """1 + popcount((row-1) xor (col-1)) (engine.py:165-170)."""
    if block_row < 1 or block_col < 1:
        raise OutOfRange("block coordinates are 1-based")
    return 1 + bin((block_row - 1) ^ (block_col - 1)).count("1")


# ---------------------------------------------------------------------------
# blocked products (engine.py:178-249) -- the block structure is validated as
# in the reference; the product itself is one K1 launch.
# ---------------------------------------------------------------------------


def _offsets(sizes) -> tuple:
    out = [0]
    for s in sizes:
        out.append(out[-1] + s)
    return tuple(out)


class BlockedView:
    """A dense array with block row/col boundaries (engine.py:178-192)."""

    __slots__ = ("data", "row_sizes", "col_sizes", "row_offsets", "col_offsets")

    def __init__(self, data, row_sizes, col_sizes):
        self.data = data
        self.row_sizes = tuple(row_sizes)
        self.col_sizes = tuple(col_sizes)
        self.row_offsets = _offsets(self.row_sizes)
        self.col_offsets = _offsets(self.col_sizes)
        if tuple(data.shape) != (self.row_offsets[-1], self.col_offsets[-1]):
            raise BlockShapeMismatch(
                f"data {tuple(data.shape)} vs block sizes {self.row_sizes} x {self.col_sizes}"
            )


def fox_block_multiply(a: BlockedView, b: BlockedView, out: BlockedView, workers: int = 1,
                       negate: bool = False, accumulate: bool = False,
                       counters: OpCounters | None = None) -> None:
    """out = (+-1) a @ b blockwise (engine.py:202-249).  The reference's Fox
    stage order is a CPU scheduling device; on the B200 the blocked product is
    a single K1 launch (block structure checked, result identical up to
    summation order)."""
    from .core import multiply

    if a.col_sizes != b.row_sizes:
        raise BlockShapeMismatch(f"a cols {a.col_sizes} vs b rows {b.row_sizes}")
    if out.row_sizes != a.row_sizes or out.col_sizes != b.col_sizes:
        raise BlockShapeMismatch(
            f"out {out.row_sizes} x {out.col_sizes} for product {a.row_sizes} x {b.col_sizes}"
        )
    multiply(a.data, b.data, out.data, accumulate=accumulate, negate=negate)
    if counters is not None:
        counters.multiplies += 1
        if accumulate:
            counters.reductions += 1


def assemble_updown(level: int, minv, t_sets: dict, workers: int = 1,
                    counters: OpCounters | None = None) -> None:
    """One assembly pass ``level`` on its own (engine.py:460-479, the step
    interpreter's ``updown_pass``, :396-437): for every level-``level`` quad
    with completed half-width diagonal inverses in ``minv``,
    M_inv[D rows, A cols] = L . M_inv[A, A] and M_inv[A rows, D cols] =
    R . M_inv[D, D], L and R taken from ``t_sets[level]``.  ``minv`` is a
    BlockMatrix or a MemoryBlockStore and is updated in place.  On the device
    the pass is two K1 products per quad (the reference's per-block-column
    tasks are one GEMM each here); ``workers`` is accepted for signature
    parity."""
    from .core import device_gemm

    store = minv.store if isinstance(minv, BlockMatrix) else minv
    scheme = store.scheme
    if level not in t_sets:
        raise BlockShapeMismatch(f"no provisional set for level {level}")
    tset = t_sets[level]
    if not 1 <= level <= scheme.k:
        raise BlockShapeMismatch(f"level {level} for {scheme.n_blocks} blocks")
    resolve_workers(workers)
    off = scheme.offsets
    quads = []
    for g in range(scheme.n_blocks >> level):  # load every operand first (MissingProvisionalData)
        first, mid, last = tset.spans(g)
        quads.append((off[first], off[mid], off[last], tset.l_block(g), tset.r_block(g)))
    dm = _lib.to_device(store.data)
    for a0, a1, a2, lb, rb in quads:
        device_gemm(_lib.to_device(lb), dm[a0:a1, a0:a1], dm[a1:a2, a0:a1])  # down: L . M_inv[A, A]
        device_gemm(_lib.to_device(rb), dm[a1:a2, a1:a2], dm[a0:a1, a1:a2])  # up:   R . M_inv[D, D]
        if counters is not None:
            counters.multiplies += 2
    out = _lib.to_numpy(dm[:, : scheme.m_n])
    for a0, a1, a2, _, _ in quads:
        store.data[a1:a2, a0:a1] = out[a1:a2, a0:a1]
        store.data[a0:a1, a1:a2] = out[a0:a1, a1:a2]


# ---------------------------------------------------------------------------
# the device engine
# ---------------------------------------------------------------------------


# Device schedules (include/blockinv_b200.h): "eq7" is the reference step
# engine (default; step/state parity); "pivot_a" is the 2n^3 block-level
# invertor_by_a recursion, one step, no stop_after_step.
SCHEDULES = {"eq7": 0, "pivot_a": 1}


class DeviceEngine:
    """A bound native engine (``bi_engine``) for one partition and batch size,
    with its device buffers: M and M_inv as [batch, n, ld] float64 tensors and
    the workspace holding every provisional set and the leaf scratch."""

    def __init__(self, sizes, batch: int = 1, schedule: str = "eq7"):
        t = _lib.torch()
        _lib.require_device()
        if schedule not in SCHEDULES:
            raise ValueError(f"schedule must be one of {sorted(SCHEDULES)}, got {schedule!r}")
        self.scheme = partition_from_sizes(sizes)
        self.sizes = tuple(int(s) for s in sizes)
        self.batch = int(batch)
        self.schedule = schedule
        self.n = self.scheme.m_n
        L = _lib.lib()
        h = _lib._vp()
        arr = (_lib._c_i64 * len(self.sizes))(*self.sizes)
        _lib.check(L.bi_engine_create_ex(_lib.ctypes.byref(h), len(self.sizes), arr, self.batch,
                                         SCHEDULES[schedule]), "bi_engine_create_ex")
        self._h = h
        self.M = _lib.empty_matrix(self.n, self.n, batch=self.batch)
        self.Minv = _lib.empty_matrix(self.n, self.n, batch=self.batch)
        self.ws = _lib.workspace(L.bi_engine_workspace_bytes(h))
        self.device = self.M.device
        with t.cuda.device(self.device):
            _lib.check(L.bi_engine_bind(h, _lib.ptr(self.M), _lib.ld(self.M), int(self.M.stride(0)),
                                        _lib.ptr(self.Minv), _lib.ld(self.Minv), int(self.Minv.stride(0)),
                                        _lib.ptr(self.ws), self.ws.numel(), _lib.stream_ptr()),
                       "bi_engine_bind")
        self.n_steps = total_steps(len(self.sizes)) if schedule == "eq7" else 1

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().bi_engine_destroy(h)
            except Exception:  # interpreter teardown
                pass
            self._h = None

    def load(self, ms, non_blocking: bool = False) -> None:
        """Copy the batch of input matrices (host array or tensor) into M."""
        t = _lib.torch()
        src = ms if isinstance(ms, t.Tensor) else t.from_numpy(np.ascontiguousarray(ms, dtype=np.float64))
        if src.dim() == 2:
            src = src.unsqueeze(0)
        if tuple(src.shape) != (self.batch, self.n, self.n):
            raise DimensionMismatch(f"input {tuple(src.shape)} vs engine ({self.batch}, {self.n}, {self.n})")
        self.M.copy_(src, non_blocking=non_blocking)

    def run(self, first: int = 1, last: int | None = None, use_graph: bool = True) -> None:
        """Enqueue steps [first, last]; M_inv is zeroed before step 1
        (storage.fresh_state, storage.py:391-411)."""
        last = self.n_steps if last is None else last
        if not 1 <= first <= last <= self.n_steps:
            raise OutOfRange(f"steps {first}..{last} outside 1..{self.n_steps}")
        if first == 1:
            self.Minv.zero_()
        rc = _lib.lib().bi_engine_run(self._h, first, last, 1 if use_graph else 0, _lib.stream_ptr())
        _lib.check(rc, "bi_engine_run")

    def run_host(self, ms: np.ndarray | None, out: np.ndarray | None, first: int = 1, last: int | None = None,
                 use_graph: bool = True) -> None:
        """End-to-end on HOST buffers (``bi_engine_run_host``): per-matrix
        host->device copies of ``ms`` [batch, n, n] overlap the other matrices'
        compute, and every inverse is copied into ``out`` [batch, n, n] as soon
        as its lane finishes.  Float64, unit column stride; page-locked buffers
        are captured into the step graph.  Asynchronous: call ``check()``."""
        last = self.n_steps if last is None else last
        n = self.n

        def spec(a, what):
            if a is None:
                return None, 0, 0
            if a.dtype != np.float64 or a.ndim not in (2, 3) or a.strides[-1] != 8:
                raise DimensionMismatch(f"{what}: float64 array with unit column stride required")
            a3 = a if a.ndim == 3 else a[None]
            if a3.shape != (self.batch, n, n):
                raise DimensionMismatch(f"{what} {a.shape} vs engine ({self.batch}, {n}, {n})")
            return a3.ctypes.data, a3.strides[1] // 8, a3.strides[0] // 8

        pi, ldi, si = spec(ms, "input")
        po, ldo, so = spec(out, "output")
        if po is not None and not out.flags.writeable:
            raise DimensionMismatch("output array is read-only")
        rc = _lib.lib().bi_engine_run_host(self._h, pi, ldi, si, po, ldo, so, first, last,
                                           1 if use_graph else 0, _lib.stream_ptr())
        _lib.check(rc, "bi_engine_run_host")

    def run_phase(self, mask: int, first: int = 1, last: int | None = None) -> None:
        """Enqueue only the K1 GEMM ops (mask 1) or only the leaf inversions
        (mask 2) of steps [first, last] -- per-kernel timing for the roofline."""
        last = self.n_steps if last is None else last
        _lib.check(_lib.lib().bi_engine_run_phase(self._h, first, last, mask, _lib.stream_ptr()),
                   "bi_engine_run_phase")

    def launches(self, first: int = 1, last: int | None = None) -> dict:
        last = self.n_steps if last is None else last
        out = (_lib._c_i64 * 3)()
        _lib.check(_lib.lib().bi_engine_launches(self._h, first, last, out), "bi_engine_launches")
        return {"total": int(out[0]), "gemm": int(out[1]), "inversion": int(out[2])}

    def check(self) -> None:
        """Synchronize; raise SingularBlock(step, quad) for the first singular
        leaf of the executed range (engine.py:320-328)."""
        s, q, z = _lib.ctypes.c_int(), _lib.ctypes.c_int(), _lib.ctypes.c_int()
        rc = _lib.lib().bi_engine_status(self._h, _lib.ctypes.byref(s), _lib.ctypes.byref(q),
                                         _lib.ctypes.byref(z))
        if _lib.check(rc, "bi_engine_status") == _lib.BI_ESINGULAR:
            exc = SingularBlock("A", path=[], step=s.value, quad=q.value)
            exc.matrix = z.value
            raise exc

    def counters(self, first: int = 1, last: int | None = None) -> dict:
        last = self.n_steps if last is None else last
        out = (_lib.ctypes.c_double * 6)()
        _lib.check(_lib.lib().bi_engine_counters(self._h, first, last, out), "bi_engine_counters")
        return {"multiplies": int(out[0]), "inversions": int(out[1]), "reductions": int(out[2]),
                "gemm_flops": out[3], "leaf_flops": out[4], "gemm_bytes": out[5]}

    def tset_square(self, level: int, quad: int, matrix: int = 0):
        """Device view of the level-`level` provisional square of a quad."""
        p, ld, side = _lib._vp(), _lib._c_i64(), _lib._c_i64()
        _lib.check(_lib.lib().bi_engine_tset_square(self._h, level, quad, matrix, _lib.ctypes.byref(p),
                                                    _lib.ctypes.byref(ld), _lib.ctypes.byref(side)),
                   "bi_engine_tset_square")
        t = _lib.torch()
        # the square lives inside self.ws: build a strided view over it
        base = _lib.ptr(self.ws)
        off = (p.value - base)
        assert off % 8 == 0 and off >= 0
        flat = self.ws.view(t.float64)
        return flat.as_strided((side.value, side.value), (ld.value, 1), off // 8)


    # --- step-boundary state (checkpoint/resume) -------------------
    def tset_levels_after(self, stepid: int) -> list[int]:
        """Levels whose provisional entries exist after ``stepid`` (the
        arrows step at level l stores every quad's L, R, S_D, S_A)."""
        nb = len(self.sizes)
        lv = set()
        for st in range(1, stepid + 1):
            a = decode_step(loopid_for_step(st, nb))
            if a.sid is not None:
                lv.add(a.sid)
        return sorted(lv)

    def _quad_spans(self, level: int, quad: int):
        off = self.scheme.offsets
        first = quad << level
        mid = first + (1 << (level - 1))
        last = (quad + 1) << level
        return off[mid] - off[first], off[last] - off[mid]

    def snapshot(self, stepid: int, matrix: int = 0):
        """(M_inv dense, {level: {(kind, idx): array}}) of one matrix after
        ``stepid`` -- the state the reference checkpoints (storage.py:292-328)."""
        if self.schedule != "eq7":
            raise ValueError("step-boundary state exists for the Eq. 7 schedule only")
        t = _lib.torch()

        def to_host(dev):  # DMA into page-locked memory (torch's caching host allocator), one sync at the end
            host = t.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
            host.copy_(dev, non_blocking=True)
            return host

        minv_h = to_host(self.Minv[matrix, :, : self.n])
        squares = {}
        for level in self.tset_levels_after(stepid):
            for g in range(len(self.sizes) >> level):
                squares[(level, g)] = to_host(self.tset_square(level, g, matrix))
        t.cuda.current_stream().synchronize()
        minv = minv_h.numpy()
        tsets = {}
        for level in self.tset_levels_after(stepid):
            entries = {}
            for g in range(len(self.sizes) >> level):
                ha, hd = self._quad_spans(level, g)
                sq = squares[(level, g)].numpy()
                # views into the page-locked copy (serialised contiguously when written)
                entries[("L", g)] = sq[ha:, :ha]
                entries[("R", g)] = sq[:ha, ha:]
                entries[("S", 2 * g)] = sq[:ha, :ha]
                entries[("S", 2 * g + 1)] = sq[ha:, ha:]
            tsets[level] = entries
        return minv, tsets

    def restore(self, minv: np.ndarray, tsets: dict, matrix: int = 0) -> None:
        """Upload a step-boundary state (inverse of ``snapshot``)."""
        t = _lib.torch()
        if self.schedule != "eq7":
            raise ValueError("step-boundary state exists for the Eq. 7 schedule only")
        self.Minv[matrix, :, : self.n].copy_(t.from_numpy(np.array(minv, dtype=np.float64)))
        for level, entries in tsets.items():
            for g in range(len(self.sizes) >> level):
                ha, hd = self._quad_spans(level, g)
                sq = self.tset_square(level, g, matrix)
                for (kind, idx), rows, cols in ((("L", g), slice(ha, None), slice(0, ha)),
                                                (("R", g), slice(0, ha), slice(ha, None)),
                                                (("S", 2 * g), slice(0, ha), slice(0, ha)),
                                                (("S", 2 * g + 1), slice(ha, None), slice(ha, None))):
                    if (kind, idx) in entries:
                        sq[rows, cols].copy_(t.from_numpy(np.array(entries[(kind, idx)], dtype=np.float64)))
        t.cuda.synchronize()


_ENGINES: "OrderedDict[tuple, DeviceEngine]" = OrderedDict()
_CACHE_MAX = 2


def _engine_for(sizes, batch: int, schedule: str = "eq7") -> DeviceEngine:
    t = _lib.torch()
    key = (tuple(int(s) for s in sizes), int(batch), schedule,
           t.cuda.current_device() if t.cuda.is_available() else -1)
    eng = _ENGINES.get(key)
    if eng is None:
        eng = DeviceEngine(sizes, batch, schedule)
        _ENGINES[key] = eng
        while len(_ENGINES) > _CACHE_MAX:
            _ENGINES.popitem(last=False)
    else:
        _ENGINES.move_to_end(key)
    return eng


def _scheme_and_dense(m, sizes):
    if isinstance(m, BlockMatrix):
        scheme = m.scheme
        if sizes is not None and tuple(int(s) for s in sizes) != scheme.sizes:
            raise SchemeMismatch("explicit sizes differ from the BlockMatrix scheme")
        return scheme, m.store.data if hasattr(m.store, "data") else m.to_dense()
    dense = np.asarray(m, dtype=np.float64)
    if dense.ndim != 2 or dense.shape[0] != dense.shape[1]:
        raise DimensionMismatch(f"square matrix required, got {dense.shape}")
    scheme = partition_from_sizes(sizes) if sizes is not None else make_partition(dense.shape[0])
    if scheme.m_n != dense.shape[0]:
        raise DimensionMismatch(f"sizes sum to {scheme.m_n}, matrix order is {dense.shape[0]}")
    return scheme, dense


def _last_step(n_steps: int, stop_after_step) -> int:
    if stop_after_step is None:
        return n_steps
    return max(1, min(int(stop_after_step), n_steps))


# --- host buffers -------------------------------------------------------------
# Pageable NumPy input goes to bi_engine_run_host as is: the engine stages it
# through its own page-locked buffer in need order, level by level, under
# the compute (bi_engine.cu run_host_pipelined).  Results up to
# _PINNED_RESULT_LIMIT bytes are allocated page-locked (torch's caching host
# allocator; the NumPy result keeps the block alive), so the inverse is
# DMA'd straight into the caller's array during the last step.
_PINNED_RESULT_LIMIT = 8 << 30


def _result_array(shape) -> np.ndarray:
    nbytes = 8 * int(np.prod(shape))
    if nbytes <= _PINNED_RESULT_LIMIT:
        t = _lib.torch()
        try:
            return t.empty(tuple(shape), dtype=t.float64, pin_memory=True).numpy()
        except RuntimeError:  # page-locked memory exhausted: pageable result
            pass
    return np.empty(shape)


def _page_locked(a: np.ndarray) -> bool:
    t = _lib.torch()
    try:
        return bool(t.from_numpy(a).is_pinned())
    except (RuntimeError, ValueError, TypeError):
        return False


def _run_host_staged(eng, src: np.ndarray, out: np.ndarray, last: int) -> None:
    """eng.run_host on host buffers (page-locked or pageable; the native
    engine pipelines pageable input in need order)."""
    eng.run_host(src, out, 1, last)
    eng.check()


def release_engines() -> None:
    """Drop the cached device engines (their M, M_inv, T-sets and page-locked
    staging) -- e.g. before a different large problem."""
    _ENGINES.clear()
    t = _lib.torch()
    if t.cuda.is_available():
        t.cuda.synchronize()
        t.cuda.empty_cache()


def gpus_for_workers(workers: int | None, nblocks: int) -> int:
    """``workers`` -> GPU count: clamped to the visible GPUs,
    then the largest power of two that also divides the block count."""
    if workers is None or workers <= 1:
        return 1
    t = _lib.torch()
    visible = t.cuda.device_count() if t.cuda.is_available() else 1
    p = 1
    while p * 2 <= min(workers, visible) and nblocks % (p * 2) == 0:
        p *= 2
    return p


def _add_counters(counters: OpCounters, sizes, last: int) -> None:
    """Reference OpCounters of steps 1..last (bi_engine_counters; no device needed)."""
    L = _lib.lib()
    h = _lib._vp()
    arr = (_lib._c_i64 * len(sizes))(*sizes)
    _lib.check(L.bi_engine_create(_lib.ctypes.byref(h), len(sizes), arr, 1), "bi_engine_create")
    try:
        out = (_lib.ctypes.c_double * 6)()
        _lib.check(L.bi_engine_counters(h, 1, last, out), "bi_engine_counters")
    finally:
        L.bi_engine_destroy(h)
    counters.multiplies += int(out[0])
    counters.inversions += int(out[1])
    counters.reductions += int(out[2])


def _check_schedule(schedule: str, stop_after_step) -> None:
    if schedule not in SCHEDULES:
        raise ValueError(f"schedule must be one of {sorted(SCHEDULES)}, got {schedule!r}")
    if schedule != "eq7" and stop_after_step is not None:
        raise ValueError("stop_after_step addresses the Eq. 7 step schedule; use schedule='eq7'")


def run_inversion(m, workers: int | None = None, checkpoint_dir=None, file_backed: bool = False,
                  sizes=None, stop_after_step: int | None = None,
                  counters: OpCounters | None = None, *, schedule: str = "eq7") -> BlockMatrix:
    """Invert a partitioned matrix through the full step schedule on the B200
    (engine.py:482-542).  Same arguments and result type as the reference;
    ``checkpoint_dir`` / ``file_backed`` (step-boundary persistence) are
    handled in the reference's on-disk format (checkpoint.py).
    Extension: ``schedule="pivot_a"`` runs the same partition through the 2n^3
    block-level pivot-A recursion (invertor_by_a, recursive.py:83-123) instead
    of the Eq. 7 steps; counters then follow invertor_by_a."""
    workers = resolve_workers(workers)
    _check_schedule(schedule, stop_after_step)
    if file_backed and checkpoint_dir is None:
        raise ValueError("file-backed mode needs a checkpoint directory")  # storage.py:396-397
    scheme, dense = _scheme_and_dense(m, sizes)
    if checkpoint_dir is not None:
        if schedule != "eq7":
            raise ValueError("checkpoints hold Eq. 7 step-boundary state; use schedule='eq7'")
        return _run_checkpointed(scheme, np.ascontiguousarray(dense, dtype=np.float64), checkpoint_dir,
                                 file_backed, stop_after_step, counters)
    gpus = gpus_for_workers(workers, len(scheme.sizes)) if schedule == "eq7" else 1
    if gpus > 1:  # column-sharded over this process's GPUs, one thread per GPU
        from .distributed import run_inversion_local

        last = _last_step(total_steps(len(scheme.sizes)), stop_after_step)
        out = run_inversion_local(np.ascontiguousarray(dense, dtype=np.float64), list(scheme.sizes), gpus,
                                  stop_after_step=last)
        if counters is not None:
            _add_counters(counters, scheme.sizes, last)
        return BlockMatrix(scheme, MemoryBlockStore(scheme, out), role="inverse")
    eng = _engine_for(scheme.sizes, 1, schedule)
    last = _last_step(eng.n_steps, stop_after_step)
    dense = np.ascontiguousarray(dense, dtype=np.float64)
    out = _result_array((scheme.m_n, scheme.m_n))
    _run_host_staged(eng, dense, out, last)
    if counters is not None:
        c = eng.counters(1, last)
        counters.multiplies += c["multiplies"]
        counters.inversions += c["inversions"]
        counters.reductions += c["reductions"]
    return BlockMatrix(scheme, MemoryBlockStore(scheme, out), role="inverse")


def _run_checkpointed(scheme, dense, directory, file_backed, stop_after_step, counters) -> BlockMatrix:
    """engine.py:515-542 with the device engine: resume a matching
    checkpoint, then after every step snapshot M_inv and the stored
    provisional entries into ``directory`` (reference format, checkpoint.py).
    ``file_backed`` keeps the reference's directory semantics (stale block
    files are dropped on a fresh start); the working state stays in HBM."""
    from . import checkpoint as ckpt

    sizes = list(scheme.sizes)
    input_hash = ckpt.input_fingerprint(dense, sizes)
    n_steps = total_steps(len(sizes))
    eng = _engine_for(scheme.sizes, 1)
    eng.load(dense)
    start = 1
    minv = None
    if ckpt.has_checkpoint(directory):
        meta = ckpt.checkpoint_load(directory)
        ckpt.checkpoint_matches(meta, sizes, input_hash)
        minv, tsets = ckpt.load_state(directory, sizes)
        eng.restore(minv, tsets)
        start = meta["stepid"] + 1
    elif file_backed:
        ckpt.clear_state(directory)
    last = n_steps if stop_after_step is None else min(n_steps, max(start, int(stop_after_step)))
    writer = ckpt.CheckpointWriter()  # checkpoint_save's files, unchanged blocks not rewritten
    for stepid in range(start, last + 1):
        eng.run(stepid, stepid, use_graph=False)
        eng.check()
        minv, tsets = eng.snapshot(stepid)
        writer.save(directory, sizes, minv, tsets, stepid, input_hash)
    if counters is not None and start <= last:
        c = eng.counters(start, last)
        counters.multiplies += c["multiplies"]
        counters.inversions += c["inversions"]
        counters.reductions += c["reductions"]
    if minv is None:  # fresh start with nothing to run cannot happen (n_steps >= 1)
        minv = eng.Minv[0, :, : eng.n].cpu().numpy()
    return BlockMatrix(scheme, MemoryBlockStore(scheme, np.array(minv)), role="inverse")


def run_inversion_batch(ms, sizes, out: np.ndarray | None = None,
                        stop_after_step: int | None = None,
                        counters: OpCounters | None = None, *, schedule: str = "eq7") -> np.ndarray:
    """Batched extension: invert ``ms`` [batch, n, n] (shared partition
    ``sizes``) in lock-step; returns (or fills ``out``) [batch, n, n].
    Page-locked ``ms``/``out`` make the host<->device copies asynchronous DMA."""
    if isinstance(ms, np.ndarray) and ms.dtype == np.float64 and ms.ndim == 3 and ms.strides[-1] == 8:
        ms_np = ms
    else:
        t = _lib.torch()
        ms_np = ms.cpu().numpy() if isinstance(ms, t.Tensor) else np.ascontiguousarray(ms, dtype=np.float64)
        ms_np = np.ascontiguousarray(ms_np, dtype=np.float64)
    if ms_np.ndim != 3 or ms_np.shape[1] != ms_np.shape[2]:
        raise DimensionMismatch(f"expected [batch, n, n], got {ms_np.shape}")
    scheme = partition_from_sizes(sizes)
    if scheme.m_n != ms_np.shape[1]:
        raise DimensionMismatch(f"sizes sum to {scheme.m_n}, matrix order is {ms_np.shape[1]}")
    _check_schedule(schedule, stop_after_step)
    eng = _engine_for(scheme.sizes, int(ms_np.shape[0]), schedule)
    last = _last_step(eng.n_steps, stop_after_step)
    if out is None:
        out = _result_array(ms_np.shape)
    _run_host_staged(eng, ms_np, out, last)
    if counters is not None:
        c = eng.counters(1, last)
        counters.multiplies += c["multiplies"]
        counters.inversions += c["inversions"]
        counters.reductions += c["reductions"]
    return out
