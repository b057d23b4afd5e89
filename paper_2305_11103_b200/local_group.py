"""In-process "process group" for the sharded engine: P threads, one per GPU,
exchanging column slabs by peer copies (NVLink) instead of NCCL.

``run_inversion(m, workers=P)`` uses it so a single Python process drives P
GPUs with the same column-sharded level schedule as the one-process-per-GPU
path (distributed.py): the reference's ``workers`` argument becomes
the GPU count (engine.py:58-65, 482-490).  The facade implements exactly the
torch.distributed calls ShardedEngine makes; every exchange is
synchronous (producer stream synchronized, barrier, peer copies, barrier), and
a failing thread aborts the barriers so the others raise instead of hanging.
"""

from __future__ import annotations

import threading
from types import SimpleNamespace


class _Group:
    def __init__(self, members: tuple[int, ...]):
        self.members = members
        self.barrier = threading.Barrier(len(members))
        self.slots: list = [None] * len(members)


class LocalWorld:
    """Shared state of one P-thread run."""

    def __init__(self, size: int):
        self.size = size
        self._lock = threading.Lock()
        self._groups: dict[tuple[int, ...], _Group] = {}
        self.world = self.group_for(tuple(range(size)))

    def group_for(self, members: tuple[int, ...]) -> _Group:
        with self._lock:
            g = self._groups.get(members)
            if g is None:
                g = self._groups[members] = _Group(members)
            return g

    def abort(self) -> None:
        with self._lock:
            for g in self._groups.values():
                g.barrier.abort()

    def facade(self, rank: int) -> "LocalDist":
        return LocalDist(self, rank)


class LocalDist:
    """The torch.distributed subset used by ShardedEngine, for thread ``rank``."""

    class ReduceOp:
        MIN = "min"

    def __init__(self, world: LocalWorld, rank: int):
        self.world = world
        self.rank = rank
        self.group = SimpleNamespace(WORLD=world.world)

    # -- topology ---------------------------------------------------------------
    def get_world_size(self, group=None) -> int:
        return len((group or self.world.world).members)

    def get_rank(self, group=None) -> int:
        return (group or self.world.world).members.index(self.rank)

    def get_global_rank(self, group, group_rank: int) -> int:
        return group.members[group_rank]

    def new_group(self, members) -> _Group:
        return self.world.group_for(tuple(int(m) for m in members))

    def get_backend(self, group=None) -> str:
        return "local"

    # -- exchanges --------------------------------------------------------------
    def _exchange(self, group: _Group, value):
        import torch

        if torch.is_tensor(value) and value.is_cuda:
            torch.cuda.current_stream(value.device).synchronize()  # producer done
        me = group.members.index(self.rank)
        group.slots[me] = value
        group.barrier.wait()
        return me, list(group.slots)

    def all_gather_into_tensor(self, recv, send, group=None) -> None:
        import torch

        group = group or self.world.world
        _, slots = self._exchange(group, send)
        for i, part in enumerate(slots):
            recv[i].copy_(part, non_blocking=recv.is_cuda)  # peer copy into this thread's device
        if recv.is_cuda:
            torch.cuda.current_stream(recv.device).synchronize()
        group.barrier.wait()  # every receiver done before any sender reuses its buffer

    def share(self, value, group=None) -> list:
        """Fused-exchange hand-off (K1P): publish ``value`` (device views) and
        return every member's, in member order, once every producer stream is
        done.  Readers access the peers' memory directly (peer access over
        NVLink); must be paired with ``release``."""
        import torch

        group = group or self.world.world
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()  # producer done
        _, slots = self._exchange(group, value)
        return slots

    def release(self, group=None) -> None:
        """Every reader's kernels done before any owner reuses its buffers."""
        import torch

        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()
        (group or self.world.world).barrier.wait()

    def all_gather(self, parts, tensor, group=None) -> None:
        group = group or self.world.world
        _, slots = self._exchange(group, tensor)
        for i, part in enumerate(slots):
            parts[i].copy_(part)
        group.barrier.wait()

    def all_reduce(self, tensor, op=None, group=None) -> None:
        import torch

        group = group or self.world.world
        _, slots = self._exchange(group, tensor.clone())
        vals = torch.stack([s.to(tensor.device) for s in slots])
        tensor.copy_(vals.min(dim=0).values if op in (None, "min") else vals.sum(dim=0))
        group.barrier.wait()


def run_threads(size: int, target, devices=None):
    """Run ``target(dist_facade, rank)`` on ``size`` threads (thread r on
    ``devices[r]``, default cuda:r); returns the per-rank results and re-raises
    the first exception."""
    import torch

    world = LocalWorld(size)
    devices = list(range(size)) if devices is None else list(devices)
    results: list = [None] * size
    errors: list = [None] * size

    def body(r: int) -> None:
        try:
            if torch.cuda.is_available() and devices[r] is not None:  # None: host-only rank (tests)
                torch.cuda.set_device(devices[r])
            results[r] = target(world.facade(r), r)
        except BaseException as exc:  # noqa: BLE001 -- surfaced below
            errors[r] = exc
            world.abort()

    threads = [threading.Thread(target=body, args=(r,), name=f"bi-gpu{r}") for r in range(size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    primary = [e for e in errors if e is not None and not isinstance(e, threading.BrokenBarrierError)]
    if primary:
        raise primary[0]
    if any(e is not None for e in errors):
        raise next(e for e in errors if e is not None)
    return results
