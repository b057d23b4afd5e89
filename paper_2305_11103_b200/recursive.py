"""Recursive blockwise inversion on the B200 (recursive.py:72-496).

The reference recurses Eq. 2 down to 2x2 analytic leaves.  On the device the
same pivot-A recursion (split floor(n/2), six products and two reductions per
node) stops at ``LEAF_ORDER`` and inverts the leaves with the K3 pivoted
Gauss-Jordan kernel -- one native call, ``bi_inplace_by_a``, for the whole
tree.  The counters report the executed tree (nodes, 6 multiplies and 2
reductions per node, one inversion per leaf).

``invertor_by_ad`` (both diagonal pivots per node, Eq. 7) recurses on device
tensors: the (A, D) and (S_D, S_A) pairs of a node whose halves are leaves
are inverted by one batched K3 call, the four products and two Schur
reductions are K1 launches, and leaf status is checked once at the end (no
host sync inside the tree).  ``invertor_with_fallback`` keeps the
reference's per-node A -> D -> B -> C pivot fallback, each node's formula on
the device.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import OpCounters, as_matrix, device_gemm, device_inverse
from .errors import AllPivotsSingular, DimensionMismatch, ScratchTooSmall, SingularBlock

LEAF_ORDER = 256  # device leaf order (the reference recurses to 2, recursive.py:44)

# ---------------------------------------------------------------------------
# OpCounters: the reference recursion's tallies.  The device executes a
# shallower tree (K3 leaves of order <= LEAF_ORDER), but the counters are an
# API contract (test_acceptance.py:112-143, test_recursive.py): they are
# computed here by replaying the reference recursion's bookkeeping -- leaf
# order 2, split floor(n/2), the same alloc/release sequence (peak_scratch)
# and the Schur workspace pool (schur_scratch) -- without its arithmetic.
# device_tree_counters() gives the executed tree's tallies.
# ---------------------------------------------------------------------------
REF_LEAF_ORDER = 2  # recursive.py:44
_REF_LIST_MAX = 10  # recursive.py:69 (list path below this order, inlined bookkeeping)


def _ref_by_a(n: int, c: OpCounters) -> None:
    """_by_a_rec / _by_a_small (recursive.py:83-123, 228-263)."""
    if n <= _REF_LIST_MAX:
        c.alloc(n * n)
        if n <= REF_LEAF_ORDER:
            c.inversions += 1
            return
        c.nodes += 1
        p, q = n // 2, n - n // 2
        _ref_by_a(p, c)
        c.alloc(2 * p * q + q * q)
        c.multiplies += 3
        c.reductions += 1
        _ref_by_a(q, c)
        c.release(q * q)
        c.multiplies += 3
        c.reductions += 1
        c.release(p * q + p * p + q * p + q * q)
        return
    c.alloc(n * n)
    c.nodes += 1
    p, q = n // 2, n - n // 2
    _ref_by_a(p, c)
    c.alloc(p * q)
    c.multiplies += 1  # n_ab = -A^-1 B
    c.alloc(q * p)
    c.multiplies += 1  # ca = C A^-1
    c.alloc(q * q)
    c.multiplies += 1  # S_A = D + C n_ab
    c.reductions += 1
    _ref_by_a(q, c)
    c.release(q * q)
    c.multiplies += 1  # out01
    c.release(p * q)
    c.release(p * p)
    c.multiplies += 1  # out00 += out01 ca
    c.reductions += 1
    c.multiplies += 1  # out10
    c.release(q * p)
    c.release(q * q)


def _ref_inplace(n: int, c: OpCounters) -> None:
    """_inplace_rec (recursive.py:317-333): 6 in-place products per node."""
    if n <= REF_LEAF_ORDER:
        c.inversions += 1
        return
    c.nodes += 1
    _ref_inplace(n // 2, c)
    c.multiplies += 3  # inplace_left, multiply(acc), inplace_right
    c.reductions += 1
    _ref_inplace(n - n // 2, c)
    c.multiplies += 3
    c.reductions += 1


def _ref_by_ad(n: int, start: int, pool: set, c: OpCounters) -> None:
    """_by_ad_rec with the _SchurPool (recursive.py:340-462)."""
    if n <= REF_LEAF_ORDER:
        c.inversions += 1
        return
    c.nodes += 1
    p, q = n // 2, n - n // 2
    c.alloc(p * p + q * q)
    _ref_by_ad(p, start, pool, c)
    _ref_by_ad(q, start + p, pool, c)
    c.alloc(p * q + q * p)
    c.multiplies += 2
    c.release(p * p + q * q)
    for key, order in (((start, p, "sd"), p), ((start + p, q, "sa"), q)):
        if key not in pool:
            pool.add(key)
            c.schur_scratch += order * order
            c.alloc(order * order)
        c.reductions += 1  # schur_accumulate
    _ref_by_ad(p, start, pool, c)
    _ref_by_ad(q, start + p, pool, c)
    c.multiplies += 2
    c.release(p * q + q * p)


def device_tree_counters(n: int, procedure: str = "by_a") -> OpCounters:
    """Tallies of the tree the device actually executes (K3 leaves of order
    <= LEAF_ORDER): pivot-A nodes carry 6 products + 2 reductions, Eq. 7
    nodes 4 + 2."""
    c = OpCounters()
    per = (4, 2) if procedure == "by_ad" else (6, 2)

    def rec(m: int) -> None:
        if m <= LEAF_ORDER:
            c.inversions += 1
            return
        c.nodes += 1
        c.multiplies += per[0]
        c.reductions += per[1]
        for _ in range(2 if procedure == "by_ad" else 1):  # Eq. 7: A, D then S_D, S_A
            rec(m // 2)
            rec(m - m // 2)

    if n:
        rec(n)
    return c


def _check_square(x) -> np.ndarray:
    x = as_matrix(x)
    if x.shape[0] != x.shape[1]:
        raise DimensionMismatch(f"need a square matrix, got {x.shape}")
    return x


def inplace_by_a_device(x_dev, leaf_order: int = LEAF_ORDER) -> None:
    """x_dev <- x_dev^-1 in place on the device (pivot-A recursion, K3 leaves)."""
    L = _lib.lib()
    n = int(x_dev.shape[0])
    ws = _lib.workspace(L.bi_inplace_by_a_workspace_bytes(n, leaf_order))
    path = _lib.ctypes.create_string_buffer(64)
    rc = L.bi_inplace_by_a(n, _lib.ptr(x_dev), _lib.ld(x_dev), leaf_order, _lib.ptr(ws), ws.numel(), path,
                           _lib.stream_ptr())
    if _lib.check(rc, "bi_inplace_by_a") == _lib.BI_ESINGULAR:
        labels = {"A": "A", "S": "SchurA"}
        raise SingularBlock("A", path=[labels[ch] for ch in path.value.decode()])


def invertor_inplace_by_a(x, row_scratch=None, counters: OpCounters | None = None) -> OpCounters:
    """Overwrite ``x`` with its inverse (recursive.py:273-292).  The
    row-scratch contract is validated as in the reference
    (ScratchTooSmall); the device recursion keeps its temporaries in HBM."""
    x = _check_square(x)
    n = x.shape[0]
    if row_scratch is None:
        row_scratch = np.empty(n)
    if row_scratch.shape[0] < n:
        raise ScratchTooSmall(f"need {n} scalars, have {row_scratch.shape[0]}")
    counters = counters if counters is not None else OpCounters()
    if n:
        xd = _lib.to_device(x)
        inplace_by_a_device(xd)
        _lib.download(xd, x)
    counters.alloc(row_scratch.shape[0])  # recursive.py:289-291
    if n:
        _ref_inplace(n, counters)
    counters.release(row_scratch.shape[0])
    return counters


def invertor_by_a(x, counters: OpCounters | None = None):
    """Pivot-A recursion into new storage (recursive.py:72-80); returns
    ``(inverse, counters)`` and leaves the input untouched."""
    x = _check_square(x)
    counters = counters if counters is not None else OpCounters()
    n = x.shape[0]
    out = np.empty((n, n))
    if n:
        xd = _lib.to_device(x)
        inplace_by_a_device(xd)
        _lib.download(xd, out)
        _ref_by_a(n, counters)
    return out, counters


# ---------------------------------------------------------------------------
# invertor_by_ad (recursive.py:366-449)
# ---------------------------------------------------------------------------


class _AdTree:
    """Device Eq. 7 recursion state: pending leaf status and the reference's
    tallies (nodes, 4 multiplies + 2 reductions per node, one inversion per
    leaf, Schur workspaces pooled per (position, order, side))."""

    def __init__(self, counters: OpCounters, leaf_order: int):
        self.counters = counters
        self.leaf_order = leaf_order
        self.pending = []  # (device info tensor, [paths])
        self.pool = {}

    def slot(self, start: int, order: int, side: str, like):
        key = (start, order, side)
        if key not in self.pool:
            self.pool[key] = _lib.empty_matrix(order, order)
            self.counters.schur_scratch += order * order
        return self.pool[key]

    def leaves(self, pairs):
        """Invert [(block, out, path)] (all leaves); equal orders share one
        K3 launch."""
        by_order = {}
        for blk, out, path in pairs:
            by_order.setdefault(int(blk.shape[0]), []).append((blk, out, path))
        for n, items in by_order.items():
            if len(items) == 1:
                blk, out, path = items[0]
                self.pending.append((device_inverse(blk, out, sync=False), [path]))
            else:
                from .core import device_inverse_list

                info = device_inverse_list([b for b, _, _ in items], [o for _, o, _ in items])
                self.pending.append((info, [p for _, _, p in items]))
            self.counters.inversions += len(items)

    def pair(self, x1, o1, s1, p1, x2, o2, s2, p2):
        """Invert two independent blocks (a reference 'pair' stage)."""
        leaf1, leaf2 = x1.shape[0] <= self.leaf_order, x2.shape[0] <= self.leaf_order
        if leaf1 and leaf2:
            self.leaves([(x1, o1, p1), (x2, o2, p2)])
            return
        for x, o, st, p, lf in ((x1, o1, s1, p1, leaf1), (x2, o2, s2, p2, leaf2)):
            if lf:
                self.leaves([(x, o, p)])
            else:
                self.node(x, o, st, p)

    def node(self, x, out, start: int, path):
        n = int(x.shape[0])
        if n <= self.leaf_order:
            self.leaves([(x, out, path)])
            return
        self.counters.nodes += 1
        p, q = n // 2, n - n // 2
        a, b, c, d = x[:p, :p], x[:p, p:], x[p:, :p], x[p:, p:]
        a_inv, d_inv = _lib.empty_matrix(p, p), _lib.empty_matrix(q, q)
        self.pair(a, a_inv, start, path + ["A"], d, d_inv, start + p, path + ["D"])
        n_ab, n_dc = _lib.empty_matrix(p, q), _lib.empty_matrix(q, p)
        device_gemm(a_inv, b, n_ab, negate=True)  # -A^-1 B
        device_gemm(d_inv, c, n_dc, negate=True)  # -D^-1 C
        s_d = self.slot(start, p, "sd", a)
        s_d.copy_(a)
        device_gemm(b, n_dc, s_d, c=s_d)  # S_D = A - B D^-1 C
        s_a = self.slot(start + p, q, "sa", d)
        s_a.copy_(d)
        device_gemm(c, n_ab, s_a, c=s_a)  # S_A = D - C A^-1 B
        self.pair(s_d, out[:p, :p], start, path + ["SchurD"], s_a, out[p:, p:], start + p, path + ["SchurA"])
        device_gemm(n_ab, out[p:, p:], out[:p, p:])  # -A^-1 B S_A^-1
        device_gemm(n_dc, out[:p, :p], out[p:, :p])  # -D^-1 C S_D^-1
        self.counters.multiplies += 4
        self.counters.reductions += 2

    def check(self) -> None:
        """Raise for the first singular leaf in execution order."""
        for info, paths in self.pending:
            bad = np.nonzero(info.cpu().numpy())[0]
            if bad.size:
                raise SingularBlock("A", path=paths[int(bad[0])])


def invertor_by_ad(x, counters: OpCounters | None = None, parallel_pairs: bool = False):
    """Both diagonal pivots per node (recursive.py:366-385); returns
    ``(inverse, counters)``.  Pairs are always independent on the device
    (batched leaves), so ``parallel_pairs`` changes nothing, as in the
    reference where results are identical either way."""
    x = _check_square(x)
    counters = counters if counters is not None else OpCounters()
    n = x.shape[0]
    out = np.empty((n, n))
    if n:
        tree = _AdTree(OpCounters(), LEAF_ORDER)  # device tree tallies: device_tree_counters
        xd = _lib.to_device(x)
        od = _lib.empty_matrix(n, n)
        tree.node(xd, od, 0, [])
        tree.check()
        _lib.download(od, out)
        _ref_by_ad(n, 0, set(), counters)
    return out, counters


# ---------------------------------------------------------------------------
# invertor_with_fallback (recursive.py:470-496)
# ---------------------------------------------------------------------------


def invertor_with_fallback(x, counters: OpCounters | None = None):
    """Recursive inversion trying pivots A, D, B, C at every node
    (recursive.py:470-496); returns ``(inverse, counters)``.  Nodes above
    ``LEAF_ORDER`` run the reference's per-node fallback
    (schur.invert_with_fallback with this recursion as ``invert_sub``, each
    product on the device); leaves use the pivoted K3 kernel, which already
    handles permutation-like blocks."""
    from .core import invert_small
    from .schur import invert_with_fallback

    x = _check_square(x)
    counters = counters if counters is not None else OpCounters()

    def leaf(block, out):
        dm = _lib.to_device(as_matrix(block))
        do = _lib.empty_matrix(*dm.shape)
        if int(device_inverse(dm, do)[0]):
            raise SingularBlock("A", path=[])
        _lib.download(do, out)
        counters.inversions += 1

    def sub(block, out):
        n = block.shape[0]
        if n <= LEAF_ORDER:
            if n <= 4:
                invert_small(block, out, counters)
            else:
                leaf(block, out)
            return
        counters.nodes += 1
        try:
            invert_with_fallback(block, n // 2, out, invert_sub=sub, counters=counters)
        except AllPivotsSingular:
            raise SingularBlock("AllPivots", path=[]) from None

    out = np.empty_like(x)
    if x.shape[0]:
        sub(x, out)
    return out, counters
