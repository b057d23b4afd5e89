"""Recursive pivot-A inversion on the B200 (recursive.py:72-333).

The reference recurses Eq. 2 down to 2x2 analytic leaves.  On the device the
same pivot-A recursion (split floor(n/2), six products and two reductions per
node) stops at ``LEAF_ORDER`` and inverts the leaves with the K3 pivoted
Gauss-Jordan kernel -- one native call, ``bi_inplace_by_a``, for the whole
tree.  The counters report the executed tree (nodes, 6 multiplies and 2
reductions per node, one inversion per leaf).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import OpCounters, as_matrix
from .errors import DimensionMismatch, ScratchTooSmall, SingularBlock

LEAF_ORDER = 256  # device leaf order (reference: 2, recursive.py:44)


def _check_square(x) -> np.ndarray:
    x = as_matrix(x)
    if x.shape[0] != x.shape[1]:
        raise DimensionMismatch(f"need a square matrix, got {x.shape}")
    return x


def _tree(n: int, leaf: int, c: OpCounters) -> None:
    if n <= leaf:
        c.inversions += 1
        return
    c.nodes += 1
    c.multiplies += 6
    c.reductions += 2
    _tree(n // 2, leaf, c)
    _tree(n - n // 2, leaf, c)


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
        x[...] = xd.cpu().numpy()
    _tree(n, LEAF_ORDER, counters)
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
        out[...] = xd.cpu().numpy()
    _tree(n, LEAF_ORDER, counters)
    return out, counters
