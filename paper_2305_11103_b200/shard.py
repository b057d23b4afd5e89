"""Native column-sharded engine over the C ABI.

``NativeShard`` is rank r of P: a ``bi_engine_create_shard`` engine whose M
and M_inv are the rank's block-column slabs (n x w) and whose schedule is the
reference's step schedule (engine.py:73-162) restricted to the home range,
with one *exchange* before every global-level action (include/blockinv_b200.h).
Every step between two exchanges is one cached CUDA graph.

Two drivers:

* ``run_group`` -- all P ranks in this process (``run_inversion(workers=P)``,
  one GPU per rank; tests put several ranks on one GPU): one native call,
  ``bi_shard_group_run``, enqueues every rank's segments and does each
  exchange as peer copies (NVLink) ordered by CUDA events.  No host barrier,
  no host sync, no Python per op.
* ``NativeShard.run_dist`` -- one process per GPU: per exchange, pack ->
  ``all_gather_into_tensor`` inside the rank group (NCCL over NVLink; gloo
  staged through host for CPU-side tests) -> unpack, all stream-ordered.

Both are bitwise equal to the single-GPU engine: GEMMs are split by output
columns only, so every output element sums the same products in the same
order for every P (the GPU analogue of test_acceptance.py:146-156).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .engine import total_steps
from .errors import DimensionMismatch, InvalidOrder, SingularBlock
from .partition import partition_from_sizes

BI_SHARD_STAGING = 1


class NativeShard:
    """Rank ``rank`` of ``nranks`` on the current CUDA device."""

    def __init__(self, sizes, nranks: int, rank: int, staging: bool = False):
        t = _lib.torch()
        self.device = _lib.require_device()
        self.scheme = partition_from_sizes(sizes)
        self.sizes = tuple(int(s) for s in self.scheme.sizes)
        nb = len(self.sizes)
        if nranks < 1 or nranks & (nranks - 1) or nb % nranks:
            raise InvalidOrder(f"{nranks} ranks must be a power of two dividing {nb} blocks")
        self.P, self.rank = int(nranks), int(rank)
        self.n = self.scheme.m_n
        self.n_steps = total_steps(nb)
        L = _lib.lib()
        h = _lib._vp()
        arr = (_lib._c_i64 * nb)(*self.sizes)
        _lib.check(L.bi_engine_create_shard(ctypes.byref(h), nb, arr, self.P, self.rank,
                                            BI_SHARD_STAGING if staging else 0), "bi_engine_create_shard")
        self._h = h
        info = (_lib._c_i64 * 8)()
        _lib.check(L.bi_engine_shard_info(h, info), "bi_engine_shard_info")
        self.c0, self.w, self.wmax = int(info[2]), int(info[3]), int(info[4])
        self.M = _lib.empty_matrix(self.n, self.w, batch=1)
        self.Minv = _lib.empty_matrix(self.n, self.w, batch=1)
        self.ws = _lib.workspace(L.bi_engine_workspace_bytes(h))
        with t.cuda.device(self.device):
            _lib.check(L.bi_engine_bind(h, _lib.ptr(self.M), _lib.ld(self.M), int(self.M.stride(0)),
                                        _lib.ptr(self.Minv), _lib.ld(self.Minv), int(self.Minv.stride(0)),
                                        _lib.ptr(self.ws), self.ws.numel(), _lib.stream_ptr()), "bi_engine_bind")
        _lib.check(L.bi_engine_shard_info(h, info), "bi_engine_shard_info")  # exchanges exist once bound
        self.n_xchg = int(info[5])
        self._segs = {}
        self._x = [self.xchg_desc(i) for i in range(self.n_xchg)]
        if staging:
            sp, rp = _lib._vp(), _lib._vp()
            _lib.check(L.bi_engine_shard_buffers(h, ctypes.byref(sp), ctypes.byref(rp)), "bi_engine_shard_buffers")
            flat = self.ws.view(t.float64)
            base = _lib.ptr(self.ws)
            self._send_off = (sp.value - base) // 8
            self._recv_off = (rp.value - base) // 8
            self._flat = flat

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().bi_engine_destroy(h)
            except Exception:  # interpreter teardown
                pass
            self._h = None

    # -- plan ------------------------------------------------------------------
    def xchg_desc(self, i: int) -> dict:
        out = (_lib._c_i64 * 8)()
        _lib.check(_lib.lib().bi_engine_xchg_desc(self._h, i, out), "bi_engine_xchg_desc")
        return {"g0": int(out[0]), "gs": int(out[1]), "rows": int(out[2]), "wmax": int(out[3]),
                "in_a": bool(out[4]), "from": (int(out[5]), int(out[6])), "kind": "arrows" if out[7] < 100 else "updown",
                "level": int(out[7]) % 100}

    def segments(self, first: int = 1, last: int | None = None) -> list[tuple[int, int, int]]:
        """[(op_begin, op_end, exchange index or -1)] of steps [first, last]."""
        last = self.n_steps if last is None else last
        key = (first, last)
        if key not in self._segs:
            L = _lib.lib()
            n = L.bi_engine_shard_segments(self._h, first, last, None, None, None, 0)
            if n < 0:
                _lib.check(n, "bi_engine_shard_segments")
            b, e, x = ((ctypes.c_int * n)() for _ in range(3))
            L.bi_engine_shard_segments(self._h, first, last, b, e, x, n)
            self._segs[key] = [(b[i], e[i], x[i]) for i in range(n)]
        return self._segs[key]

    # -- data ------------------------------------------------------------------
    def load(self, m) -> None:
        """This rank's column slab of the full host matrix ``m``."""
        t = _lib.torch()
        m = np.asarray(m)
        if m.shape != (self.n, self.n):
            raise DimensionMismatch(f"matrix {m.shape} vs order {self.n}")
        self.M[0].copy_(t.from_numpy(np.ascontiguousarray(m[:, self.c0:self.c0 + self.w], dtype=np.float64)))

    def write_slab(self, out: np.ndarray) -> None:
        out[:, self.c0:self.c0 + self.w] = self.Minv[0].cpu().numpy()

    def check(self):
        """(step, block) of this rank's first singular leaf, or None (syncs)."""
        s, q, z = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        rc = _lib.lib().bi_engine_status(self._h, ctypes.byref(s), ctypes.byref(q), ctypes.byref(z))
        if _lib.check(rc, "bi_engine_status") == _lib.BI_ESINGULAR:
            return s.value, q.value
        return None

    def launches(self, first: int = 1, last: int | None = None) -> int:
        last = self.n_steps if last is None else last
        out = (_lib._c_i64 * 3)()
        _lib.check(_lib.lib().bi_engine_launches(self._h, first, last, out), "bi_engine_launches")
        return int(out[0])

    # -- one process per GPU ----------------------------------------------------
    def run_dist(self, dist, groups: dict, first: int = 1, last: int | None = None, use_graph: bool = True) -> None:
        """Steps [first, last] with the exchanges as all-gathers inside the rank
        groups (``groups[(gs, g0)]``, created by make_groups).  NCCL keeps every
        call stream-ordered (no host sync); gloo stages through host memory."""
        t = _lib.torch()
        L = _lib.lib()
        last = self.n_steps if last is None else last
        st = _lib.stream_ptr()
        if first == 1:
            self.Minv.zero_()
        for b, e, xi in self.segments(first, last):
            _lib.check(L.bi_engine_run_ops(self._h, b, e, 1 if use_graph else 0, st), "bi_engine_run_ops")
            if xi < 0:
                continue
            x = self._x[xi]
            chunk = x["rows"] * self.wmax
            _lib.check(L.bi_engine_xchg_pack(self._h, xi, st), "bi_engine_xchg_pack")
            if x["gs"] == 1:  # an up/down half of one rank: packed straight into the receive area
                _lib.check(L.bi_engine_xchg_unpack(self._h, xi, st), "bi_engine_xchg_unpack")
                continue
            send = self._flat[self._send_off:self._send_off + chunk]
            recv = self._flat[self._recv_off:self._recv_off + x["gs"] * chunk]
            pg = groups[(x["gs"], x["g0"])]
            if dist.get_backend(pg) == "nccl":
                dist.all_gather_into_tensor(recv, send, group=pg)
            else:  # gloo: through host memory (tests: several ranks on one GPU)
                parts = [t.empty(chunk, dtype=t.float64) for _ in range(x["gs"])]
                dist.all_gather(parts, send.cpu(), group=pg)
                recv.copy_(t.cat(parts).to(recv.device))
            _lib.check(L.bi_engine_xchg_unpack(self._h, xi, st), "bi_engine_xchg_unpack")


class LibNccl:
    """Transport C: NCCL inside the library (bi_nccl.cu).  The world
    communicator is created from a unique id that rank 0 draws and
    ``exchange_id`` hands to every rank (e.g. a torch.distributed
    broadcast); ``attach`` splits the group communicators of a shard."""

    def __init__(self, nranks: int, rank: int, exchange_id):
        L = _lib.lib()
        if not L.bi_nccl_available():
            raise _lib.CollectiveError("libnccl.so.2 is not loadable: no in-library NCCL transport")
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _lib.check(L.bi_nccl_unique_id(uid), "bi_nccl_unique_id")
        uid = exchange_id(bytes(uid.raw))
        self.comm = _lib._vp()
        _lib.check(L.bi_nccl_comm_init(int(nranks), uid, int(rank), ctypes.byref(self.comm)), "bi_nccl_comm_init")

    def attach(self, shard: "NativeShard") -> None:
        _lib.check(_lib.lib().bi_engine_shard_set_comm(shard._h, self.comm), "bi_engine_shard_set_comm")

    def run(self, shard: "NativeShard", first: int = 1, last: int | None = None, use_graph: bool = True) -> None:
        last = shard.n_steps if last is None else last
        _lib.check(_lib.lib().bi_engine_run_nccl(shard._h, first, last, 1 if use_graph else 0, _lib.stream_ptr()),
                   "bi_engine_run_nccl")

    def close(self) -> None:
        if self.comm.value:
            _lib.lib().bi_nccl_comm_destroy(self.comm)
            self.comm = _lib._vp()


def make_groups(dist, nranks: int, group=None) -> dict:
    """Every power-of-two rank group of the level scheduler, created
    collectively in the same order on every rank: {(size, first rank): pg}."""
    groups = {}
    gs = 2
    while gs <= nranks:
        for g0 in range(0, nranks, gs):
            members = list(range(g0, g0 + gs))
            if group is not None and group is not dist.group.WORLD:
                members = [dist.get_global_rank(group, m) for m in members]
            groups[(gs, g0)] = dist.new_group(members)
        gs *= 2
    return groups


def run_group(shards: list, first: int = 1, last: int | None = None, use_graph: bool = True,
              streams: list | None = None) -> None:
    """Steps [first, last] of all P ranks of this process in one native call
    (bi_shard_group_run; peer-copy exchanges); asynchronous on ``streams``
    (default: each shard device's current stream)."""
    t = _lib.torch()
    P = len(shards)
    last = shards[0].n_steps if last is None else last
    if streams is None:
        streams = [t.cuda.current_stream(s.device) for s in shards]
    hs = (_lib._vp * P)(*[s._h.value for s in shards])
    ss = (_lib._vp * P)(*[int(st.cuda_stream) for st in streams])
    _lib.check(_lib.lib().bi_shard_group_run(hs, P, ss, first, last, 1 if use_graph else 0), "bi_shard_group_run")


def first_singular(shards_or_results) -> tuple[int, int] | None:
    fails = [f for f in shards_or_results if f is not None]
    return min(fails) if fails else None


def run_inversion_group(m, sizes, gpus: int, stop_after_step=None, devices=None) -> np.ndarray:
    """The sharded schedule on ``gpus`` ranks of THIS process (``devices[r]``
    for rank r, default cuda:r); returns the full inverse, each rank's
    column slab copied straight into the result."""
    t = _lib.torch()
    m = np.asarray(m, dtype=np.float64)
    devices = list(range(gpus)) if devices is None else [int(d) for d in devices]
    _lib.init_devices(sorted(set(devices)))
    shards = []
    for r in range(gpus):
        with t.cuda.device(devices[r]):
            sh = NativeShard(sizes, gpus, r)
            sh.load(m)
            shards.append(sh)
    for d in set(devices):
        t.cuda.synchronize(d)
    nsteps = shards[0].n_steps
    last = nsteps if stop_after_step is None else max(1, min(int(stop_after_step), nsteps))
    run_group(shards, 1, last)
    fail = first_singular([sh.check() for sh in shards])
    if fail is not None:
        raise SingularBlock("A", path=[], step=fail[0], quad=fail[1])
    out = np.empty(m.shape)
    for sh in shards:
        sh.write_slab(out)
    return out
