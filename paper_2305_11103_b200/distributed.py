"""Multi-GPU level scheduler for the step engine: one process per
GPU, torch.distributed (NCCL over NVLink) for the exchanges.

Partitioning (engine.py:313-437): with P ranks
and N_b diagonal blocks (P | N_b), rank r owns the home range of blocks
H_r = [r N_b/P, (r+1) N_b/P) and stores *block columns* H_r of M, M_inv and of
every provisional set T_l (all rows).  The step schedule is the reference's
(stepid -> loopid -> action, engine.py:73-162), executed by every rank:

* diag (leaf inversions)  -- every leaf block lies in one home range: local;
* arrows at a local level -- the quad lies in one home range: local;
* arrows at a global level (the quad spans a rank group G = G_A u G_D): each
  rank sends its (side x w) column slab -- G_A ranks [A^-1 ; C], G_D ranks
  [B ; D^-1] -- in one all-gather inside G; G_A ranks then form their columns
  of L = -D^-1 C and S_D = A + B L, G_D ranks their columns of R = -A^-1 B and
  S_A = D + C R;
* up/down pass at a global level -- G_A ranks all-gather L, G_D ranks R,
  then each forms its columns of M_inv[D, A] = L M_inv[A, A] /
  M_inv[A, D] = R M_inv[D, D].

Every GEMM is split by output columns only (K is never split), so the
inverse is bitwise identical for every P (the GPU analogue of the reference's
worker-count determinism, test_acceptance.py:146-156).

The compute backend defaults to the B200 kernels (K1 GEMM, K3 leaf
inversion through the C ABI).  ``backend=`` accepts any object with the same
three methods; the CPU multi-process tests use that to exercise this
schedule and its collectives with the gloo backend.
"""

from __future__ import annotations

import numpy as np

from .engine import decode_step, loopid_for_step, total_steps, INVERT_DIAGONALS, ARROWS_AND_SCHUR
from .errors import DimensionMismatch, InvalidOrder, SingularBlock
from .partition import partition_from_sizes


class DeviceBackend:
    """B200 kernels through the C ABI (K1 / K3)."""

    def __init__(self):
        from . import _lib

        self._lib = _lib
        self.device = _lib.require_device()

    def empty(self, rows: int, cols: int):
        return self._lib.empty_matrix(rows, cols)

    def gemm(self, a, b, d, c=None, negate=False):
        from .core import device_gemm

        device_gemm(a, b, d, c=c, negate=negate)

    kseg_align = 16  # K1P segment boundaries lie on k-tiles

    def gemm_kseg(self, segs, b, d, c=None, negate=False):
        """K1P: d = [c] + (+-1) [segs...] @ b, segments read in place (peer GPUs)."""
        from .core import device_gemm_kseg

        device_gemm_kseg(segs, b, d, c=c, negate=negate)

    def inverse(self, blocks, outs):
        """blocks/outs: [count, b, b] strided views; returns the device info
        tensor (no host sync; checked after the run)."""
        from .core import device_inverse

        return device_inverse(blocks, outs, sync=False)

    def inverse_list(self, blocks, outs):
        """Equal-order blocks anywhere in device memory, one K3 launch chain
        (pointer tables); returns the device info tensor."""
        from .core import device_inverse_list

        return device_inverse_list(blocks, outs)


def _batched_gemms(be, products):
    """products: list of (a, b, d, c, negate) of one kind over the quads of a
    level, in quad order.  Split in one pass into maximal runs whose windows
    line up (same storage, shape and strides, constant offset step per
    operand) and issue one strided-batch launch per run: a whole level when
    the partition is uniform and the windows share a buffer, one run per
    covering T-set square otherwise."""

    def key(v):
        try:
            store = v.untyped_storage().data_ptr()
        except (AttributeError, RuntimeError):
            store = id(v)
        return (store, tuple(v.shape), tuple(v.stride())), v.storage_offset()

    n = len(products)
    ops = [[key(p[k]) if p[k] is not None else None for k in range(4)] for p in products]
    i = 0
    while i < n:
        j = i + 1
        if j < n:
            ok = all((ops[i][k] is None) == (ops[j][k] is None) for k in range(4))
            steps = [None if ops[i][k] is None else ops[j][k][1] - ops[i][k][1] for k in range(4)]
            ok = ok and all(s is None or s > 0 for s in steps)
            while ok and j < n:
                for k in range(4):
                    if ops[i][k] is None:
                        continue
                    if ops[j][k][0] != ops[i][k][0] or ops[j][k][1] - ops[j - 1][k][1] != steps[k]:
                        ok = False
                        break
                if ok:
                    j += 1
        run = products[i:j]
        if len(run) == 1:
            a, b, d, c, neg = run[0]
            be.gemm(a, b, d, c=c, negate=neg)
        else:
            def stack(k):
                v0 = run[0][k]
                return v0.as_strided((len(run),) + tuple(v0.shape), (steps[k],) + tuple(v0.stride()),
                                     v0.storage_offset())
            be.gemm(stack(0), stack(1), stack(2), c=stack(3) if run[0][3] is not None else None, negate=run[0][4])
        i = j


def _group_ranks(rank: int, group_size: int) -> list[int]:
    g0 = rank // group_size * group_size
    return list(range(g0, g0 + group_size))


class ShardedEngine:
    """One rank's share of the step engine for ``sizes`` over a process group."""

    def __init__(self, sizes, group=None, backend=None, dist=None):
        if dist is None:  # a LocalDist facade (local_group.py) drives P GPUs from one process
            import torch.distributed as dist

        self.dist = dist
        self.group = group if group is not None else dist.group.WORLD
        self.P = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.scheme = partition_from_sizes(sizes)
        self.sizes = list(self.scheme.sizes)
        self.nb = len(self.sizes)
        if self.P & (self.P - 1) or self.nb % self.P:
            raise InvalidOrder(f"{self.P} ranks must be a power of two dividing {self.nb} blocks")
        self.off = list(self.scheme.offsets)
        self.n = self.scheme.m_n
        self.k = self.nb.bit_length() - 1
        self.nbp = self.nb // self.P  # blocks per rank
        self.h0 = self.rank * self.nbp
        self.h1 = self.h0 + self.nbp
        self.c0 = self.off[self.h0]
        self.w = self.off[self.h1] - self.c0
        self.be = backend if backend is not None else DeviceBackend()
        # Fused exchange (K1P): with an in-process group whose members can read
        # each other's memory (local_group.py, peer access over NVLink) and a
        # backend with gemm_kseg, global-level GEMMs read the peers' column
        # slabs in place instead of all-gathering them first.
        import os

        # Opt-in (BI_FUSED_GATHER=1): K1 re-reads each A row block once per
        # 64-column tile, so at the K1 rate the in-place form needs ~2 TB/s of
        # peer reads (0.5 TB/s with a 4-CTA multicast cluster) against 0.9 TB/s
        # per NVLink 5 direction, while the gathered copy costs ~4 % of the
        # GEMM it feeds (DESIGN 7, profiles/r01_kseg_fused_gather.txt).
        self.fused = (hasattr(dist, "share") and hasattr(self.be, "gemm_kseg")
                      and os.environ.get("BI_FUSED_GATHER", "0") == "1")
        # column-slab storage
        self.M = self.be.empty(self.n, self.w)
        self.Minv = self.be.empty(self.n, self.w)
        self.T = {}
        for lv in range(1, self.k + 1):
            shapes = {}
            for g in range(self.nb >> lv):
                first, last = g << lv, (g + 1) << lv
                if last <= self.h0 or first >= self.h1:
                    continue
                side = self.off[last] - self.off[first]
                cols = self.off[min(last, self.h1)] - self.off[max(first, self.h0)]
                shapes[g] = (side, cols)
            if len(set(shapes.values())) == 1:  # equal quads: one stacked buffer (batchable windows)
                side, cols = next(iter(shapes.values()))
                buf = self.be.empty(side * len(shapes), cols)
                for i, g in enumerate(sorted(shapes)):
                    self.T[(lv, g)] = buf[i * side:(i + 1) * side]
            else:
                for g, (side, cols) in shapes.items():
                    self.T[(lv, g)] = self.be.empty(side, cols)
        # rank groups for the global levels (created collectively, same order everywhere)
        self.groups = {}
        world_ranks = list(range(self.P))
        gs = 2
        while gs <= self.P:
            for g0 in range(0, self.P, gs):
                members = world_ranks[g0:g0 + gs]
                pg = dist.new_group([dist.get_global_rank(self.group, m) for m in members]) \
                    if self.group is not dist.group.WORLD else dist.new_group(members)
                if self.rank in members:
                    self.groups[gs] = pg
            gs *= 2

    # -- layout helpers -----------------------------------------------------
    def is_global(self, level: int) -> bool:
        return (1 << level) > self.nbp

    def _cols(self, c0: int, c1: int) -> tuple[int, int]:
        if c0 < self.h0 or c1 > self.h1:
            raise IndexError(f"block columns {c0}:{c1} not on rank {self.rank}")
        return self.off[c0] - self.c0, self.off[c1] - self.c0

    def m_win(self, r0, r1, c0, c1):
        a, b = self._cols(c0, c1)
        return self.M[self.off[r0]:self.off[r1], a:b]

    def minv_win(self, r0, r1, c0, c1):
        a, b = self._cols(c0, c1)
        return self.Minv[self.off[r0]:self.off[r1], a:b]

    def t_win(self, level, r0, r1, c0, c1):
        g = min(r0, c0) >> level
        sq = self.T[(level, g)]
        o = self.off[g << level]
        col_origin = max(self.off[g << level], self.c0)
        a = self.off[c0] - col_origin
        b = self.off[c1] - col_origin
        return sq[self.off[r0] - o:self.off[r1] - o, a:b]

    def src_win(self, act, r0, r1, c0, c1):
        if act.source == "matrix":
            return self.m_win(r0, r1, c0, c1)
        return self.t_win(act.cid, r0, r1, c0, c1)

    # -- step actions -------------------------------------------------------
    def _diag(self, act, stepid):
        blocks = list(range(self.h0, self.h1))
        if hasattr(self.be, "inverse_list"):  # every equal-order leaf of the step in one call
            by_size = {}
            for p in blocks:
                by_size.setdefault(self.sizes[p], []).append(p)
            for b, ps in by_size.items():
                src = [self.src_win(act, p, p + 1, p, p + 1) for p in ps]
                dst = [self.minv_win(p, p + 1, p, p + 1) for p in ps]
                self._infos.append((stepid, ps, self.be.inverse_list(src, dst)))
            return
        # group runs of equal-size consecutive blocks inside one buffer
        runs, cur = [], [blocks[0]]
        for p in blocks[1:]:
            same_buf = act.source == "matrix" or (p >> act.cid) == (cur[0] >> act.cid)
            if self.sizes[p] == self.sizes[cur[0]] and same_buf:
                cur.append(p)
            else:
                runs.append(cur)
                cur = [p]
        runs.append(cur)
        for run in runs:
            b = self.sizes[run[0]]
            src0 = self.src_win(act, run[0], run[0] + 1, run[0], run[0] + 1)
            dst0 = self.minv_win(run[0], run[0] + 1, run[0], run[0] + 1)
            cnt = len(run)
            src = src0.as_strided((cnt, b, b), (b * (src0.stride(0) + 1), src0.stride(0), 1))
            dst = dst0.as_strided((cnt, b, b), (b * (dst0.stride(0) + 1), dst0.stride(0), 1))
            self._infos.append((stepid, run, self.be.inverse(src, dst)))  # resolved in check()

    def _quad(self, level, g):
        first = g << level
        mid = first + (1 << (level - 1))
        return first, mid, (g + 1) << level

    def _allgather_tensor(self, send, pg, size):
        """[size, *send.shape] all-gather: NCCL device-to-device; gloo (CPU
        tests, or several ranks sharing one GPU) stages through host memory."""
        import torch

        send = send.contiguous()
        if self.dist.get_backend(pg) in ("nccl", "local"):
            recv = torch.empty((size,) + tuple(send.shape), dtype=send.dtype, device=send.device)
            self.dist.all_gather_into_tensor(recv, send, group=pg)
            return recv
        host = send.cpu()
        parts = [torch.empty_like(host) for _ in range(size)]
        self.dist.all_gather(parts, host, group=pg)
        return torch.stack(parts).to(send.device)

    def _width(self, r: int) -> int:
        return self.off[(r + 1) * self.nbp] - self.off[r * self.nbp]

    def _allgather(self, level, slab):
        """All-gather column slabs inside this rank's level-`level` group; slabs
        are padded to the group's widest home range and trimmed on receipt."""
        import torch

        gs = (1 << level) // self.nbp
        members = _group_ranks(self.rank, gs)
        wmax = max(self._width(m) for m in members)
        if slab.shape[1] < wmax:
            padded = torch.zeros((slab.shape[0], wmax), dtype=slab.dtype, device=slab.device)
            padded[:, :slab.shape[1]] = slab
            slab = padded
        recv = self._allgather_tensor(slab, self.groups[gs], gs)
        return [recv[i][:, :self._width(m)] for i, m in enumerate(members)], members

    def _fusable(self, lv, act, in_a) -> bool:
        """K1P applies when the owners' slab widths put every segment boundary
        on a k-tile, the group has at most 8 owners per half, and no shared
        slab is overwritten by this level's outputs (sources other than T_lv)."""
        if not self.fused:
            return False
        if act is not None and act.source != "matrix" and act.cid == lv:
            return False
        gs = (1 << lv) // self.nbp
        members = _group_ranks(self.rank, gs)
        if gs // 2 > 8:
            return False
        align = getattr(self.be, "kseg_align", 1)
        half = [m for m in members if (self._rank_h1(m) <= self._quad(lv, self.h0 >> lv)[1]) == in_a]
        other = [m for m in members if m not in half]
        return all(self._width(m) % align == 0 for grp in (half, other) for m in grp[:-1])

    def _share(self, level, value):
        """Publish this rank's slab views inside its level group; returns every
        member's views (producer streams done) and the member ranks."""
        gs = (1 << level) // self.nbp
        return self.dist.share(value, group=self.groups[gs]), _group_ranks(self.rank, gs)

    def _release(self, level):
        """Every member done reading before any owner overwrites a shared slab."""
        self.dist.release(group=self.groups[(1 << level) // self.nbp])

    def _arrows(self, act):
        lv = act.sid
        be = self.be
        if not self.is_global(lv):
            # all local quads of the level at once: R and L, then S_D and S_A
            # (one strided-batch launch per product when the quads are equal-sized)
            r_ops, l_ops, sd_ops, sa_ops = [], [], [], []
            for g in range(self.h0 >> lv, self.h1 >> lv):
                first, mid, last = self._quad(lv, g)
                A = self.src_win(act, first, mid, first, mid)
                B = self.src_win(act, first, mid, mid, last)
                C = self.src_win(act, mid, last, first, mid)
                D = self.src_win(act, mid, last, mid, last)
                R = self.t_win(lv, first, mid, mid, last)
                L = self.t_win(lv, mid, last, first, mid)
                r_ops.append((self.minv_win(first, mid, first, mid), B, R, None, True))
                l_ops.append((self.minv_win(mid, last, mid, last), C, L, None, True))
                sd_ops.append((B, L, self.t_win(lv, first, mid, first, mid), A, False))
                sa_ops.append((C, R, self.t_win(lv, mid, last, mid, last), D, False))
            for ops in (r_ops, l_ops, sd_ops, sa_ops):
                _batched_gemms(be, ops)
            return
        import torch

        g = self.h0 >> lv
        first, mid, last = self._quad(lv, g)
        in_a = self.h1 <= mid
        ha = self.off[mid] - self.off[first]
        # my slab: A-half ranks send [A^-1 ; C] cols, D-half ranks [B ; D^-1] cols
        mine = (self.h0, self.h1)
        if in_a:
            top = self.minv_win(first, mid, *mine)
            bot = self.src_win(act, mid, last, *mine)
        else:
            top = self.src_win(act, first, mid, *mine)
            bot = self.minv_win(mid, last, *mine)
        if self._fusable(lv, act, in_a):
            # peers' A^-1 / B / C / D^-1 column slabs are K segments of K1P, read in place
            shared, members = self._share(lv, (top, bot))
            peers = [i for i, m in enumerate(members) if (self._rank_h1(m) <= mid) != in_a]
            tops, bots = [shared[i][0] for i in peers], [shared[i][1] for i in peers]
            if in_a:  # L = -D^-1 C, S_D = A + B L (my columns)
                L_my = self.t_win(lv, mid, last, *mine)
                self.be.gemm_kseg(bots, self.src_win(act, mid, last, *mine), L_my, negate=True)
                self.be.gemm_kseg(tops, L_my, self.t_win(lv, first, mid, *mine), c=self.src_win(act, first, mid, *mine))
            else:     # R = -A^-1 B, S_A = D + C R (my columns)
                R_my = self.t_win(lv, first, mid, *mine)
                self.be.gemm_kseg(tops, self.src_win(act, first, mid, *mine), R_my, negate=True)
                self.be.gemm_kseg(bots, R_my, self.t_win(lv, mid, last, *mine), c=self.src_win(act, mid, last, *mine))
            self._release(lv)
            return
        slab = torch.cat([top, bot], dim=0)
        recv, members = self._allgather(lv, slab)
        peers = [i for i, m in enumerate(members) if (self._rank_h1(m) <= mid) != in_a]
        top_full = torch.cat([recv[i][:ha] for i in peers], dim=1)   # A^-1 or B
        bot_full = torch.cat([recv[i][ha:] for i in peers], dim=1)   # C or D^-1
        if in_a:
            B, Dinv = top_full, bot_full
            C_my = self.src_win(act, mid, last, *mine)
            A_my = self.src_win(act, first, mid, *mine)
            L_my = self.t_win(lv, mid, last, *mine)
            self.be.gemm(Dinv, C_my, L_my, negate=True)
            self.be.gemm(B, L_my, self.t_win(lv, first, mid, *mine), c=A_my)
        else:
            Ainv, C = top_full, bot_full
            B_my = self.src_win(act, first, mid, *mine)
            D_my = self.src_win(act, mid, last, *mine)
            R_my = self.t_win(lv, first, mid, *mine)
            self.be.gemm(Ainv, B_my, R_my, negate=True)
            self.be.gemm(C, R_my, self.t_win(lv, mid, last, *mine), c=D_my)

    def _rank_h1(self, r):
        return (r + 1) * self.nbp

    def _updown(self, lv):
        be = self.be
        if not self.is_global(lv):
            down, up = [], []
            for g in range(self.h0 >> lv, self.h1 >> lv):
                first, mid, last = self._quad(lv, g)
                down.append((self.t_win(lv, mid, last, first, mid), self.minv_win(first, mid, first, mid),
                             self.minv_win(mid, last, first, mid), None, False))
                up.append((self.t_win(lv, first, mid, mid, last), self.minv_win(mid, last, mid, last),
                           self.minv_win(first, mid, mid, last), None, False))
            _batched_gemms(be, down)
            _batched_gemms(be, up)
            return
        import torch

        g = self.h0 >> lv
        first, mid, last = self._quad(lv, g)
        in_a = self.h1 <= mid
        mine = (self.h0, self.h1)
        ha, hd = self.off[mid] - self.off[first], self.off[last] - self.off[mid]
        hmax = max(ha, hd)
        # A-half ranks carry their L columns (C position), D-half ranks their R columns
        part = self.t_win(lv, mid, last, *mine) if in_a else self.t_win(lv, first, mid, *mine)
        if self._fusable(lv, None, in_a):
            shared, members = self._share(lv, part)
            segs = [shared[i] for i, m in enumerate(members) if (self._rank_h1(m) <= mid) == in_a]
            if in_a:  # M_inv[D, A] = L M_inv[A, A]
                be.gemm_kseg(segs, self.minv_win(first, mid, *mine), self.minv_win(mid, last, *mine))
            else:     # M_inv[A, D] = R M_inv[D, D]
                be.gemm_kseg(segs, self.minv_win(mid, last, *mine), self.minv_win(first, mid, *mine))
            self._release(lv)
            return
        slab = torch.zeros((hmax, part.shape[1]), dtype=part.dtype, device=part.device)
        slab[:part.shape[0]] = part
        recv, members = self._allgather(lv, slab)
        same = [i for i, m in enumerate(members) if (self._rank_h1(m) <= mid) == in_a]
        if in_a:
            L = torch.cat([recv[i][:hd] for i in same], dim=1)        # hd x ha
            be.gemm(L, self.minv_win(first, mid, *mine), self.minv_win(mid, last, *mine))
        else:
            R = torch.cat([recv[i][:ha] for i in same], dim=1)        # ha x hd
            be.gemm(R, self.minv_win(mid, last, *mine), self.minv_win(first, mid, *mine))

    # -- driver -------------------------------------------------------------
    def load(self, m: np.ndarray) -> None:
        """Copy this rank's column slab of the full matrix ``m``."""
        import torch

        if m.shape != (self.n, self.n):
            raise DimensionMismatch(f"matrix {m.shape} vs order {self.n}")
        self.M.copy_(torch.from_numpy(np.ascontiguousarray(m[:, self.c0:self.c0 + self.w])))

    def run(self, first: int = 1, last: int | None = None) -> None:
        nsteps = total_steps(self.nb)
        # the reference always runs at least one step and stops at N_s
        last = nsteps if last is None else max(first, min(int(last), nsteps))
        first = max(1, min(first, nsteps))
        if first == 1:
            self.Minv.zero_()
        self._first_fail = None
        self._infos = []
        for stepid in range(first, last + 1):
            act = decode_step(loopid_for_step(stepid, self.nb))
            if act.kind == INVERT_DIAGONALS:
                self._diag(act, stepid)
            elif act.kind == ARROWS_AND_SCHUR:
                self._arrows(act)
            else:
                self._diag(act, stepid)
                for lv in range(1, act.depth + 1):
                    self._updown(lv)

    def check(self) -> None:
        """Raise SingularBlock(step, quad) for the first singular leaf on any
        rank (engine.py:320-328); collective."""
        import torch

        for stepid, run, info in getattr(self, "_infos", []):
            info = info.cpu().numpy() if torch.is_tensor(info) else np.asarray(info)
            bad = np.nonzero(info)[0]
            if len(bad) and self._first_fail is None:
                self._first_fail = (stepid, run[int(bad[0])])
        self._infos = []
        mine = self._first_fail or (1 << 30, 1 << 30)
        t = torch.tensor([mine[0] * (self.nb + 1) + mine[1]], dtype=torch.int64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.to(self.M.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        v = int(t.item())
        if v < (1 << 30) * (self.nb + 1):
            raise SingularBlock("A", path=[], step=v // (self.nb + 1), quad=v % (self.nb + 1))

    def launches(self):
        """Kernel launches per run (not tracked by the host-driven engine)."""
        return None

    def write_slab(self, out: np.ndarray) -> None:
        """Copy this rank's block columns of M_inv into ``out[:, c0:c0+w]``
        (``out`` is the caller's full n x n host array, shared by the
        threads of one process)."""
        if self.w:
            out[:, self.c0:self.c0 + self.w] = self.Minv.cpu().numpy()

    def _global(self, r: int) -> int:
        if self.group is self.dist.group.WORLD:
            return r
        return self.dist.get_global_rank(self.group, r)

    def gather(self, root: int = 0):
        """The full inverse on ``root`` (None on the other ranks); collective.
        Slabs travel one at a time (root receives each into one buffer and
        writes it into its host array), so no rank ever holds more than its
        own slab plus one peer slab on the device."""
        import torch

        wmax = max(self._width(r) for r in range(self.P))
        nccl = self.dist.get_backend(self.group) == "nccl"
        dev = self.Minv.device if nccl else torch.device("cpu")
        buf = torch.zeros((self.n, wmax), dtype=self.Minv.dtype, device=dev)
        out = np.empty((self.n, self.n)) if self.rank == root else None
        for r in range(self.P):
            if r == root:
                if self.rank == root:
                    self.write_slab(out)
                continue
            wr = self._width(r)
            if self.rank == r:
                buf[:, :self.w] = self.Minv
                self.dist.send(buf, dst=self._global(root), group=self.group)
            elif self.rank == root:
                self.dist.recv(buf, src=self._global(r), group=self.group)
                c = self.off[r * self.nbp]
                out[:, c:c + wr] = buf[:, :wr].cpu().numpy()
        return out


class NativeShardDist:
    """This process's rank of the native column-sharded engine (shard.py),
    exchanging over a torch.distributed group (NCCL)."""

    def __init__(self, sizes, group=None, dist=None):
        if dist is None:
            import torch.distributed as dist
        from .shard import NativeShard, make_groups

        self.dist = dist
        self.group = group if group is not None else dist.group.WORLD
        P, rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        self.shard = NativeShard(sizes, P, rank, staging=True)
        self.P, self.rank, self.n = P, rank, self.shard.n
        self._last = self.shard.n_steps
        # BI_SHARD_TRANSPORT=lib: the exchanges as NCCL calls inside the
        # library (one C call per run); default: torch.distributed collectives
        import os

        self.lib = None
        if os.environ.get("BI_SHARD_TRANSPORT") == "lib" and dist.get_backend(self.group) == "nccl":
            from .shard import LibNccl

            def share_id(raw: bytes) -> bytes:
                box = [raw]
                dist.broadcast_object_list(box, src=dist.get_global_rank(self.group, 0)
                                           if self.group is not dist.group.WORLD else 0, group=self.group)
                return box[0]

            self.lib = LibNccl(P, rank, share_id)
            self.lib.attach(self.shard)
            self.groups = {}
        else:
            self.groups = make_groups(dist, P, self.group)

    def load(self, m) -> None:
        self.shard.load(m)

    def run(self, first: int = 1, last: int | None = None) -> None:
        nsteps = self.shard.n_steps
        last = nsteps if last is None else max(first, min(int(last), nsteps))
        self._last = last
        if self.lib is not None:
            self.lib.run(self.shard, first, last)
        else:
            self.shard.run_dist(self.dist, self.groups, first, last)

    def check(self) -> None:
        """SingularBlock(step, quad) of the earliest singular leaf on any rank (collective)."""
        import torch

        fail = self.shard.check()
        nb = len(self.shard.sizes)
        mine = fail or (1 << 30, 1 << 30)
        t = torch.tensor([mine[0] * (nb + 1) + mine[1]], dtype=torch.int64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.to(self.shard.M.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        v = int(t.item())
        if v < (1 << 30) * (nb + 1):
            raise SingularBlock("A", path=[], step=v // (nb + 1), quad=v % (nb + 1))

    def launches(self) -> int:
        return self.shard.launches(1, self._last)

    def gather(self, root: int = 0):
        """The full inverse on ``root`` (None elsewhere): slabs sent one at a time."""
        import torch

        sh = self.shard
        glob = (lambda r: r) if self.group is self.dist.group.WORLD else \
            (lambda r: self.dist.get_global_rank(self.group, r))
        nccl = self.dist.get_backend(self.group) == "nccl"
        buf = torch.zeros((sh.n, sh.wmax), dtype=torch.float64, device=sh.M.device if nccl else "cpu")
        out = np.empty((sh.n, sh.n)) if self.rank == root else None
        off = sh.scheme.offsets
        nbp = len(sh.sizes) // self.P
        for r in range(self.P):
            if r == root:
                if self.rank == root:
                    sh.write_slab(out)
                continue
            c0, c1 = off[r * nbp], off[(r + 1) * nbp]
            if self.rank == r:
                buf[:, :sh.w] = sh.Minv[0]
                self.dist.send(buf, dst=glob(root), group=self.group)
            elif self.rank == root:
                self.dist.recv(buf, src=glob(r), group=self.group)
                out[:, c0:c1] = buf[:, :c1 - c0].cpu().numpy()
        return out


def sharded_engine(sizes, group=None):
    """This process's rank of the column-sharded engine (one process per
    GPU, torch.distributed NCCL group): the native engine."""
    return NativeShardDist(sizes, group=group)


def run_inversion_sharded(m, sizes, group=None, backend=None, stop_after_step=None, dist=None, root: int = 0):
    """run_inversion (engine.py:482-542) with the matrix column-sharded over the
    ranks of ``group`` (one process per GPU).  Every rank passes the same
    ``m``; rank ``root`` receives the full inverse, the others None.  Raises
    SingularBlock like the single-device engine.  The native engine runs
    unless a compute ``backend`` is given (CPU tests of the schedule)."""
    if backend is None:
        eng = NativeShardDist(sizes, group=group, dist=dist)
    else:
        eng = ShardedEngine(sizes, group=group, backend=backend, dist=dist)
    eng.load(np.asarray(m, dtype=np.float64))
    eng.run(1, stop_after_step)
    eng.check()
    return eng.gather(root)


def run_inversion_local(m, sizes, gpus: int, stop_after_step=None, devices=None, backend_factory=None) -> np.ndarray:
    """The sharded schedule on ``gpus`` GPUs of THIS process.  Default: the
    native engine, all ranks driven by one native call with peer-copy
    exchanges (shard.run_inversion_group).  ``backend_factory`` (CPU tests)
    or BI_FUSED_GATHER=1 (K1P, DESIGN 7) run the host-driven ShardedEngine on
    one thread per GPU (local_group.py).  ``devices`` overrides the rank ->
    device map (tests run several ranks on one GPU)."""
    import os

    from .local_group import run_threads

    m = np.asarray(m, dtype=np.float64)
    if backend_factory is None and os.environ.get("BI_FUSED_GATHER", "0") != "1":
        from .shard import run_inversion_group

        return run_inversion_group(m, sizes, gpus, stop_after_step=stop_after_step, devices=devices)
    if backend_factory is None:  # peer access between the participating devices (bi_init)
        from . import _lib

        _lib.init_devices(sorted(set(devices if devices is not None else range(gpus))))
    out = np.empty(m.shape)

    def target(dist, rank):
        be = backend_factory() if backend_factory is not None else None
        eng = ShardedEngine(sizes, backend=be, dist=dist)
        eng.load(m)
        eng.run(1, stop_after_step)
        eng.check()
        eng.write_slab(out)  # each thread its own block columns, no all-gather

    run_threads(gpus, target, devices=devices)
    return out
