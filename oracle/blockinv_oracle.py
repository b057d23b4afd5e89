"""TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference ``blockinv`` hot path.

Every function names the reference code it restates (paths relative to
``/root/reference/pkg/src/blockinv``).  Arithmetic follows the reference's
operation order (ascending inner index, sign folded into the left factor,
CPython ``sum`` for the small list paths) so that, run in the same
interpreter, the oracle reproduces the reference bit for bit on the golden
fixtures; the tests assert this where it holds.

Errors are reported with the oracle's own light exception classes (mirrors of
``errors.py``), which the tests map onto the product's exceptions.
"""

from __future__ import annotations

import math
import operator

import numpy as np

__all__ = [
    "OracleSingular",
    "OracleSingularMatrix",
    "OracleAllPivotsSingular",
    "default_sizes",
    "offsets_of",
    "total_steps",
    "loopid_for_step",
    "decode_step",
    "updown_iteration_map",
    "mm_acc",
    "multiply",
    "invert_small",
    "gauss_jordan",
    "invertor_by_a",
    "invertor_inplace_by_a",
    "invertor_by_ad",
    "invert_via_a",
    "invert_via_d",
    "invert_via_ad",
    "invert_via_b",
    "invert_via_c",
    "invert_via_bc",
    "invert_with_fallback",
    "small_sub",
    "by_a_sub",
    "gj_sub",
    "offsets_of",
    "run_inversion",
    "EngineCounts",
    "residual_max",
    "residual_frob",
    "rel_frob",
    "lapack_inverse",
    "flops_engine",
    "pivot_a_blocks",
    "flops_pivot_a",
]


# ---------------------------------------------------------------------------
# errors (errors.py:20-38, :17-18, :41-42)
# ---------------------------------------------------------------------------


class OracleSingular(Exception):
    """Mirror of ``SingularBlock`` (errors.py:20-38): block name, path, step, quad."""

    def __init__(self, block, path=None, step=None, quad=None):
        self.block, self.path, self.step, self.quad = block, list(path or []), step, quad
        super().__init__(f"singular {block} path={self.path} step={step} quad={quad}")


class OracleSingularMatrix(Exception):
    """Mirror of ``SingularMatrix`` (errors.py:17-18), raised by the GJ oracle."""


class OracleAllPivotsSingular(Exception):
    """Mirror of ``AllPivotsSingular`` (errors.py:41-42)."""


# ---------------------------------------------------------------------------
# partition metadata (partition.py:63-99)
# ---------------------------------------------------------------------------


def default_sizes(order: int) -> list[int]:
    """Restates ``make_partition`` (partition.py:63-84): 2**(floor(log2 n)-1)
    blocks of order 2, the surplus r turning trailing blocks into 3s, then 4s."""
    if order < 2:
        raise ValueError(f"order must be >= 2, got {order}")
    nb = 2 ** max(int(math.log2(order)) - 1, 0)
    surplus = order - 2 * nb
    if surplus <= nb:
        return [2] * (nb - surplus) + [3] * surplus
    fours = surplus - nb
    return [3] * (nb - fours) + [4] * fours


def offsets_of(sizes) -> list[int]:
    """Prefix sums (partition.py:53-60 ``_build``)."""
    out = [0]
    for s in sizes:
        out.append(out[-1] + int(s))
    return out


# ---------------------------------------------------------------------------
# step schedule (engine.py:73-170)
# ---------------------------------------------------------------------------


def total_steps(nblocks: int) -> int:
    """engine.py:73-74."""
    return 2 * nblocks - 1


def loopid_for_step(stepid: int, nblocks: int) -> list[int]:
    """engine.py:77-90: descending 1-based set-bit positions, zero-padded to
    log2(nblocks)+1 entries."""
    if nblocks < 1 or nblocks & (nblocks - 1):
        raise ValueError("nblocks must be a power of two")
    if not 1 <= stepid <= total_steps(nblocks):
        raise ValueError("stepid out of range")
    width = nblocks.bit_length()
    bits = [b + 1 for b in reversed(range(width)) if (stepid >> b) & 1]
    return bits + [0] * (width - len(bits))


def decode_step(loopid) -> dict:
    """engine.py:117-157.  Returns {kind, source, cid, sid, depth} with kind in
    {"diag", "arrows", "assemble"} and source in {"matrix", "tset"}."""
    nz = [v for v in loopid if v]
    tail = list(loopid[len(nz):])
    if not nz or any(v <= 0 for v in nz) or any(tail) or any(
        a <= b for a, b in zip(nz, nz[1:])
    ):
        raise ValueError(f"malformed loopid {loopid}")
    last = nz[-1]
    if len(nz) == 1:
        if last == 1:
            return dict(kind="diag", source="matrix", cid=None, sid=None, depth=0)
        return dict(kind="arrows", source="matrix", cid=None, sid=last - 1, depth=0)
    cid = nz[-2] - 1
    if last == 1:
        # length of the trailing ..., 3, 2, 1 run
        run = 1
        while run < len(nz) and nz[-run - 1] == run + 1:
            run += 1
        return dict(kind="assemble", source="tset", cid=cid, sid=None, depth=run - 1)
    return dict(kind="arrows", source="tset", cid=cid, sid=last - 1, depth=0)


def updown_iteration_map(row: int, col: int) -> int:
    """engine.py:165-170: 1 + popcount((row-1) xor (col-1))."""
    if row < 1 or col < 1:
        raise ValueError("1-based")
    return 1 + bin((row - 1) ^ (col - 1)).count("1")


# ---------------------------------------------------------------------------
# dense kernels (core.py:107-192)
# ---------------------------------------------------------------------------

_SMALL_PRODUCT = 512  # core.py:111
_SMALL_EDGE = 8  # core.py:112


def mm_acc(a: np.ndarray, b: np.ndarray, out: np.ndarray, negate: bool = False) -> None:
    """core.py:115-139: out += (+-1)*a@b, ascending inner index, sign on a.

    Tiny products go through CPython ``sum`` (as the reference does); larger
    ones are rank-1 updates in ascending k.
    """
    m, kdim = a.shape
    n = out.shape[1]
    if m <= _SMALL_EDGE and n <= _SMALL_EDGE and m * n * kdim <= _SMALL_PRODUCT:
        rows = a.tolist()
        if negate:
            rows = [[-x for x in r] for r in rows]
        cols = list(zip(*b.tolist()))
        cur = out.tolist()
        out[...] = [
            [sum(map(operator.mul, ra, cb), o) for o, cb in zip(orow, cols)]
            for ra, orow in zip(rows, cur)
        ]
        return
    left = -a if negate else a
    scratch = np.empty_like(out)
    for k in range(kdim):
        np.multiply(left[:, k, None], b[k], out=scratch)
        np.add(out, scratch, out=out)


def multiply(a, b, out, accumulate=False, negate=False):
    """core.py:142-170 (without the alias asserts)."""
    if a.shape[1] != b.shape[0] or out.shape != (a.shape[0], b.shape[1]):
        raise ValueError("shape mismatch")
    if not accumulate:
        out[...] = 0.0
    mm_acc(a, b, out, negate)


# ---------------------------------------------------------------------------
# small analytic inverses (core.py:256-376)
# ---------------------------------------------------------------------------


def _det_tol(rows) -> float:
    """core.py:256-264: 1e-12 * n^2 * amax^n."""
    n = len(rows)
    amax = max(abs(v) for r in rows for v in r) if n else 0.0
    return 1e-12 * n * n * amax**n


def _inv2_rows(rows):
    (a, b), (c, d) = rows
    det = a * d - b * c
    if abs(det) <= _det_tol(rows):
        raise OracleSingular("A")
    r = 1.0 / det
    return [[d * r, -b * r], [-c * r, a * r]]


def _inv3_rows(rows):
    (a00, a01, a02), (a10, a11, a12), (a20, a21, a22) = rows
    k00 = a11 * a22 - a12 * a21
    k01 = -(a10 * a22 - a12 * a20)
    k02 = a10 * a21 - a11 * a20
    det = a00 * k00 + a01 * k01 + a02 * k02
    if abs(det) <= _det_tol(rows):
        raise OracleSingular("A")
    r = 1.0 / det
    k10 = -(a01 * a22 - a02 * a21)
    k11 = a00 * a22 - a02 * a20
    k12 = -(a00 * a21 - a01 * a20)
    k20 = a01 * a12 - a02 * a11
    k21 = -(a00 * a12 - a02 * a10)
    k22 = a00 * a11 - a01 * a10
    return [[k00 * r, k10 * r, k20 * r], [k01 * r, k11 * r, k21 * r], [k02 * r, k12 * r, k22 * r]]


def _inv4(m: np.ndarray, use_d: bool) -> np.ndarray:
    """core.py:300-347: 2x2-blocked pivot formula with analytic 2x2 pieces."""
    a, b, c, d = m[:2, :2], m[:2, 2:], m[2:, :2], m[2:, 2:]
    out = np.empty((4, 4))
    if use_d:
        a, d, b, c = d, a, c, b  # pivot on D: swap roles, then swap placement
    try:
        piv = np.array(_inv2_rows(a.tolist()))
    except OracleSingular:
        raise OracleSingular("D" if use_d else "A") from None
    n_pb = np.empty((2, 2))
    multiply(piv, b, n_pb, negate=True)
    cp = np.empty((2, 2))
    multiply(c, piv, cp)
    schur = d.copy()
    mm_acc(c, n_pb, schur)
    try:
        sinv = np.array(_inv2_rows(schur.tolist()))
    except OracleSingular:
        raise OracleSingular("SchurD" if use_d else "SchurA") from None
    t = np.empty((2, 2))
    multiply(n_pb, sinv, t)
    tl = piv.copy()
    multiply(t, cp, tl, accumulate=True, negate=True)
    bl = np.empty((2, 2))
    multiply(sinv, cp, bl, negate=True)
    if not use_d:
        out[:2, :2], out[:2, 2:], out[2:, :2], out[2:, 2:] = tl, t, bl, sinv
    else:
        out[2:, 2:], out[2:, :2], out[:2, 2:], out[:2, :2] = tl, t, bl, sinv
    return out


def invert_small(m: np.ndarray) -> np.ndarray:
    """core.py:350-376: closed forms for orders 1..4 (order 4 retries pivot D)."""
    n = m.shape[0]
    if m.shape != (n, n) or not 1 <= n <= 4:
        raise ValueError("invert_small needs order 1..4")
    if n == 1:
        x = float(m[0, 0])
        if x == 0.0:
            raise OracleSingular("A")
        return np.array([[1.0 / x]])
    if n == 2:
        return np.array(_inv2_rows(m.tolist()))
    if n == 3:
        return np.array(_inv3_rows(m.tolist()))
    try:
        return _inv4(m, use_d=False)
    except OracleSingular:
        return _inv4(m, use_d=True)


# ---------------------------------------------------------------------------
# Gauss-Jordan oracle (core.py:379-402)
# ---------------------------------------------------------------------------


def gauss_jordan(m: np.ndarray) -> np.ndarray:
    """core.py:379-402: partial-pivot GJ on [m | I]; a pivot column whose
    best |entry| <= 1e-12 * n * max|m| raises ``OracleSingularMatrix``."""
    m = np.asarray(m, dtype=np.float64)
    n = m.shape[0]
    if m.ndim != 2 or m.shape[1] != n:
        raise ValueError("square matrix required")
    tol = 1e-12 * n * (float(np.abs(m).max()) if m.size else 0.0)
    work = np.concatenate([m.copy(), np.eye(n)], axis=1)
    for c in range(n):
        p = c + int(np.argmax(np.abs(work[c:, c])))
        if abs(work[p, c]) <= tol:
            raise OracleSingularMatrix(f"no pivot in column {c}")
        if p != c:
            work[[c, p]] = work[[p, c]]
        work[c, :] /= work[c, c]
        f = work[:, c].copy()
        f[c] = 0.0
        work -= np.outer(f, work[c, :])
    return np.ascontiguousarray(work[:, n:])


def gj_sub(block: np.ndarray, out: np.ndarray) -> None:
    """The reference's own pivoted ``invert_sub`` injection (tests/test_schur.py:25-26)."""
    try:
        out[...] = gauss_jordan(block)
    except OracleSingularMatrix:
        raise OracleSingular("A") from None


# ---------------------------------------------------------------------------
# recursive pivot-A inversions (recursive.py:72-333)
# ---------------------------------------------------------------------------

_PY_RECURSION_MAX = 10  # recursive.py:69
_LEAF_ORDER = 2  # recursive.py:44


def _rows_mm(a, b, negate=False, start=None):
    """recursive.py:126-207 ``_mm_rows``: list product; inner <= 5 summed
    left-to-right from 0.0 (or from ``start``), wider via CPython ``sum``."""
    if negate:
        a = [[-x for x in r] for r in a]
    inner = len(b)
    cols = list(zip(*b))
    out = []
    for i, ra in enumerate(a):
        row = []
        for j, cb in enumerate(cols):
            if inner <= 5:
                acc = 0.0 if start is None else start[i][j]
                for x, y in zip(ra, cb):
                    acc = acc + x * y
            elif start is None:
                acc = sum(map(operator.mul, ra, cb))
            else:
                acc = sum(map(operator.mul, ra, cb), start[i][j])
            row.append(acc)
        out.append(row)
    return out


def _leaf_rows(rows, path):
    """recursive.py:210-225."""
    if len(rows) == 1:
        v = rows[0][0]
        if v == 0.0:
            raise OracleSingular("A", path)
        return [[1.0 / v]]
    (a, b), (c, d) = rows
    det = a * d - b * c
    amax = max(abs(a), abs(b), abs(c), abs(d))
    if abs(det) <= 1e-12 * 4 * amax * amax:
        raise OracleSingular("A", path)
    r = 1.0 / det
    return [[d * r, -b * r], [-c * r, a * r]]


def _by_a_rows(x, path):
    """recursive.py:228-265 (list path, order <= 10)."""
    n = len(x)
    if n <= _LEAF_ORDER:
        return _leaf_rows(x, path)
    p = n // 2
    a = [r[:p] for r in x[:p]]
    b = [r[p:] for r in x[:p]]
    c = [r[:p] for r in x[p:]]
    d = [r[p:] for r in x[p:]]
    ainv = _by_a_rows(a, path + ["A"])
    n_ab = _rows_mm(ainv, b, negate=True)
    ca = _rows_mm(c, ainv)
    s_a = _rows_mm(c, n_ab, start=[r[:] for r in d])
    sinv = _by_a_rows(s_a, path + ["SchurA"])
    o01 = _rows_mm(n_ab, sinv)
    o00 = _rows_mm(o01, ca, negate=True, start=[r[:] for r in ainv])
    o10 = _rows_mm(sinv, ca, negate=True)
    return [o00[i] + o01[i] for i in range(p)] + [o10[i] + sinv[i] for i in range(n - p)]


def _by_a(x: np.ndarray, path) -> np.ndarray:
    """recursive.py:83-123 (array path, order > 10)."""
    n = x.shape[0]
    if n <= _PY_RECURSION_MAX:
        return np.array(_by_a_rows(x.tolist(), path), dtype=np.float64).reshape(n, n)
    p = n // 2
    q = n - p
    a, b, c, d = x[:p, :p], x[:p, p:], x[p:, :p], x[p:, p:]
    ainv = _by_a(a, path + ["A"])
    n_ab = np.empty((p, q))
    multiply(ainv, b, n_ab, negate=True)
    ca = np.empty((q, p))
    multiply(c, ainv, ca)
    s_a = d.copy()
    multiply(c, n_ab, s_a, accumulate=True)
    sinv = _by_a(s_a, path + ["SchurA"])
    out = np.empty((n, n))
    multiply(n_ab, sinv, out[:p, p:])
    out[:p, :p] = ainv
    multiply(out[:p, p:], ca, out[:p, :p], accumulate=True, negate=True)
    multiply(sinv, ca, out[p:, :p], negate=True)
    out[p:, p:] = sinv
    return out


def invertor_by_a(x: np.ndarray) -> np.ndarray:
    """recursive.py:72-80: unpivoted recursive pivot-A inverse into new storage."""
    x = np.asarray(x, dtype=np.float64)
    return _by_a(x, [])


def _by_ad(x: np.ndarray, out: np.ndarray, path) -> None:
    """recursive.py:424-449: both diagonal pivots per node (Eq. 7), leaves of
    order <= 2 by ``invert_small``; the Schur complements are accumulated
    in place (schur_accumulate = _mm_acc into a copy of A / D)."""
    n = x.shape[0]
    if n <= 2:
        try:
            out[...] = invert_small(x)
        except OracleSingular as exc:
            raise OracleSingular(exc.block, path) from None
        return
    p = n // 2
    q = n - p
    a, b, c, d = x[:p, :p], x[:p, p:], x[p:, :p], x[p:, p:]
    ainv, dinv = np.empty((p, p)), np.empty((q, q))
    _by_ad(a, ainv, path + ["A"])
    _by_ad(d, dinv, path + ["D"])
    n_ab, n_dc = np.empty((p, q)), np.empty((q, p))
    multiply(ainv, b, n_ab, negate=True)
    multiply(dinv, c, n_dc, negate=True)
    s_d = a.copy()
    mm_acc(b, n_dc, s_d)
    s_a = d.copy()
    mm_acc(c, n_ab, s_a)
    _by_ad(s_d, out[:p, :p], path + ["SchurD"])
    _by_ad(s_a, out[p:, p:], path + ["SchurA"])
    multiply(n_ab, out[p:, p:], out[:p, p:])
    multiply(n_dc, out[:p, :p], out[p:, :p])


def invertor_by_ad(x: np.ndarray) -> np.ndarray:
    """recursive.py:366-385: combined-pivot recursion into new storage."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _by_ad(x, out, [])
    return out


def _inplace_leaf(x: np.ndarray, path) -> None:
    """recursive.py:295-314."""
    tol = _det_tol(x.tolist())
    if x.shape[0] == 1:
        v = x[0, 0]
        if abs(v) <= tol:
            raise OracleSingular("A", path)
        x[0, 0] = 1.0 / v
        return
    det = x[0, 0] * x[1, 1] - x[0, 1] * x[1, 0]
    if abs(det) <= tol:
        raise OracleSingular("A", path)
    r = 1.0 / det
    a00 = x[0, 0]
    x[0, 0] = x[1, 1] * r
    x[1, 1] = a00 * r
    x[0, 1] = -x[0, 1] * r
    x[1, 0] = -x[1, 0] * r


def _left_inplace(ainv, t, negate):
    """core.py:195-225: t <- (+-)ainv @ t, one column at a time, ascending k."""
    n = t.shape[0]
    s = np.empty(n)
    for j in range(t.shape[1]):
        col = t[:, j]
        s[:] = 0.0
        for k in range(n):
            ak = -ainv[:, k] if negate else ainv[:, k]
            s += ak * col[k]
        col[:] = s


def _right_inplace(t, ainv, negate):
    """core.py:228-253: t <- (+-)t @ ainv, one row at a time, ascending k."""
    n = t.shape[1]
    s = np.empty(n)
    for i in range(t.shape[0]):
        row = t[i, :]
        s[:] = 0.0
        for k in range(n):
            ak = -ainv[k, :] if negate else ainv[k, :]
            s += row[k] * ak
        row[:] = s


def _inplace_rec(x: np.ndarray, path) -> None:
    """recursive.py:317-333."""
    n = x.shape[0]
    if n <= _LEAF_ORDER:
        _inplace_leaf(x, path)
        return
    p = n // 2
    a, b, c, d = x[:p, :p], x[:p, p:], x[p:, :p], x[p:, p:]
    _inplace_rec(a, path + ["A"])
    _left_inplace(a, b, negate=True)
    multiply(c, b, d, accumulate=True)
    _right_inplace(c, a, negate=True)
    _inplace_rec(d, path + ["SchurA"])
    _left_inplace(d, c, negate=False)
    multiply(b, c, a, accumulate=True)
    _right_inplace(b, d, negate=False)


def invertor_inplace_by_a(x: np.ndarray) -> None:
    """recursive.py:273-292: overwrite ``x`` with its inverse."""
    _inplace_rec(x, [])


# ---------------------------------------------------------------------------
# single-level 2x2 formulas (schur.py:104-164, 219-259, 300-333)
# ---------------------------------------------------------------------------


def _sub(invert_sub, block, label):
    """schur.py:104-111."""
    out = np.empty_like(block)
    try:
        invert_sub(block, out)
    except OracleSingular as exc:
        raise OracleSingular(label, exc.path) from None
    return out


def small_sub(block, out):
    """``invert_small`` in the reference's ``invert_sub(block, out)`` protocol."""
    out[...] = invert_small(block)


def by_a_sub(block, out):
    """``invertor_by_a`` as sub-inverter (the reference's cfg3 default pattern)."""
    out[...] = invertor_by_a(block)


def invert_via_a(m: np.ndarray, split: int, invert_sub, out: np.ndarray) -> None:
    """schur.py:114-139 (Eq. 2)."""
    p = split
    a, b, c, d = m[:p, :p], m[:p, p:], m[p:, :p], m[p:, p:]
    ainv = _sub(invert_sub, a, "A")
    n_ab = np.empty_like(b)
    multiply(ainv, b, n_ab, negate=True)
    ca = np.empty_like(c)
    multiply(c, ainv, ca)
    s_a = d.copy()
    multiply(c, n_ab, s_a, accumulate=True)
    sinv = _sub(invert_sub, s_a, "SchurA")
    multiply(n_ab, sinv, out[:p, p:])
    out[:p, :p] = ainv
    multiply(out[:p, p:], ca, out[:p, :p], accumulate=True, negate=True)
    multiply(sinv, ca, out[p:, :p], negate=True)
    out[p:, p:] = sinv


def invert_via_d(m: np.ndarray, split: int, invert_sub, out: np.ndarray) -> None:
    """schur.py:142-164 (Eq. 3): pivot on D, S_D = A - B D^-1 C."""
    p = split
    a, b, c, d = m[:p, :p], m[:p, p:], m[p:, :p], m[p:, p:]
    dinv = _sub(invert_sub, d, "D")
    n_dc = np.empty_like(c)
    multiply(dinv, c, n_dc, negate=True)
    bd = np.empty_like(b)
    multiply(b, dinv, bd)
    s_d = a.copy()
    multiply(b, n_dc, s_d, accumulate=True)
    sinv = _sub(invert_sub, s_d, "SchurD")
    multiply(n_dc, sinv, out[p:, :p])
    out[p:, p:] = dinv
    multiply(out[p:, :p], bd, out[p:, p:], accumulate=True, negate=True)
    multiply(sinv, bd, out[:p, p:], negate=True)
    out[:p, :p] = sinv


def invert_via_ad(m: np.ndarray, split: int, invert_sub, out: np.ndarray) -> None:
    """schur.py:219-259 (Eq. 7): both diagonal pivots, Schur inverses on the diagonal."""
    p = split
    a, b, c, d = m[:p, :p], m[:p, p:], m[p:, :p], m[p:, p:]
    ainv = _sub(invert_sub, a, "A")
    dinv = _sub(invert_sub, d, "D")
    n_ab = np.empty_like(b)
    multiply(ainv, b, n_ab, negate=True)
    n_dc = np.empty_like(c)
    multiply(dinv, c, n_dc, negate=True)
    s_a = d.copy()
    mm_acc(c, n_ab, s_a)
    s_d = a.copy()
    mm_acc(b, n_dc, s_d)
    for blk, view, label in ((s_d, out[:p, :p], "SchurD"), (s_a, out[p:, p:], "SchurA")):
        try:
            invert_sub(blk, view)
        except OracleSingular as exc:
            raise OracleSingular(label, exc.path) from None
    multiply(n_ab, out[p:, p:], out[:p, p:])
    multiply(n_dc, out[:p, :p], out[p:, :p])


def _cquad(m, split):
    """schur.py:92-101: rows split at `split`, columns at n - split."""
    cs = m.shape[0] - split
    return m[:split, :cs], m[:split, cs:], m[split:, :cs], m[split:, cs:]


def invert_via_b(m: np.ndarray, split: int, invert_sub, out: np.ndarray) -> None:
    """schur.py:167-190: square off-diagonal pivot B, S_B = C - D B^-1 A."""
    a, b, c, d = _cquad(m, split)
    p, w = b.shape[0], c.shape[0]
    binv = _sub(invert_sub, b, "B")
    n_ba = np.empty_like(a)
    multiply(binv, a, n_ba, negate=True)
    db = np.empty_like(d)
    multiply(d, binv, db)
    s_b = c.copy()
    multiply(d, n_ba, s_b, accumulate=True)
    sinv = _sub(invert_sub, s_b, "SchurB")
    multiply(n_ba, sinv, out[w:, p:])
    out[w:, :p] = binv
    multiply(out[w:, p:], db, out[w:, :p], accumulate=True, negate=True)
    multiply(sinv, db, out[:w, :p], negate=True)
    out[:w, p:] = sinv


def invert_via_c(m: np.ndarray, split: int, invert_sub, out: np.ndarray) -> None:
    """schur.py:193-216: square off-diagonal pivot C, S_C = B - A C^-1 D."""
    a, b, c, d = _cquad(m, split)
    p, w = b.shape[0], c.shape[0]
    cinv = _sub(invert_sub, c, "C")
    n_cd = np.empty_like(d)
    multiply(cinv, d, n_cd, negate=True)
    ac = np.empty_like(a)
    multiply(a, cinv, ac)
    s_c = b.copy()
    multiply(a, n_cd, s_c, accumulate=True)
    sinv = _sub(invert_sub, s_c, "SchurC")
    multiply(n_cd, sinv, out[:w, :p])
    out[:w, p:] = cinv
    multiply(out[:w, :p], ac, out[:w, p:], accumulate=True, negate=True)
    multiply(sinv, ac, out[w:, p:], negate=True)
    out[w:, :p] = sinv


def invert_via_bc(m: np.ndarray, split: int, invert_sub, out: np.ndarray) -> None:
    """schur.py:262-297: both counter-diagonal pivots."""
    a, b, c, d = _cquad(m, split)
    p, w = b.shape[0], c.shape[0]
    binv = _sub(invert_sub, b, "B")
    cinv = _sub(invert_sub, c, "C")
    n_ba = np.empty_like(a)
    multiply(binv, a, n_ba, negate=True)
    n_cd = np.empty_like(d)
    multiply(cinv, d, n_cd, negate=True)
    s_b = c.copy()
    mm_acc(d, n_ba, s_b)
    s_c = b.copy()
    mm_acc(a, n_cd, s_c)
    for blk, view, label in ((s_b, out[:w, p:], "SchurB"), (s_c, out[w:, :p], "SchurC")):
        try:
            invert_sub(blk, view)
        except OracleSingular as exc:
            raise OracleSingular(label, exc.path) from None
    multiply(n_cd, out[w:, :p], out[:w, :p])
    multiply(n_ba, out[:w, p:], out[w:, p:])


def invert_with_fallback(m: np.ndarray, split: int, out: np.ndarray, invert_sub=None) -> str:
    """schur.py:300-333: pivots in the fixed order A, D, B, C."""
    invert_sub = invert_sub or small_sub
    errs = []
    for name, fn in (("via_a", invert_via_a), ("via_d", invert_via_d), ("via_b", invert_via_b),
                     ("via_c", invert_via_c)):
        try:
            fn(m, split, invert_sub, out)
            return name
        except OracleSingular as exc:
            errs.append(f"{name}: {exc}")
    raise OracleAllPivotsSingular("; ".join(errs))


# ---------------------------------------------------------------------------
# the 2^k-block step engine (engine.py:178-542, storage.py:166-262, 391-411)
# ---------------------------------------------------------------------------


class EngineCounts:
    """``OpCounters`` fields the engine touches (engine.py:317, 344-345, 411)."""

    def __init__(self):
        self.multiplies = 0
        self.inversions = 0
        self.reductions = 0


def _fox(a, rs_a, cs_a, b, cs_b, out, negate=False, accumulate=False):
    """engine.py:202-249: block row i accumulates its stage-t products with
    inner block (i+t) mod nb, each product through ``mm_acc``."""
    ro, ko = offsets_of(rs_a), offsets_of(cs_a)
    if not accumulate:
        out[...] = 0.0
    nbk = len(cs_a)
    for i in range(len(rs_a)):
        panel = out[ro[i]:ro[i + 1], :]
        for t in range(nbk):
            k = (i + t) % nbk
            mm_acc(a[ro[i]:ro[i + 1], ko[k]:ko[k + 1]], b[ko[k]:ko[k + 1], :], panel, negate)


def _leaf(block: np.ndarray, leaf_inverter) -> np.ndarray:
    """engine.py:449-457: <=4 analytic, else unpivoted pivot-A recursion.
    ``leaf_inverter`` overrides the >4 branch (e.g. the pivoted GJ oracle)."""
    if block.shape[0] <= 4:
        return invert_small(block)
    if leaf_inverter is not None:
        return leaf_inverter(block)
    return invertor_by_a(block)


def run_inversion(m, sizes=None, stop_after_step=None, counts=None, leaf_inverter=None,
                  return_state=False):
    """engine.py:482-542 in memory: returns the inverse under construction
    (M_inv) and, with ``return_state``, the provisional sets
    ``{level: {"L": [...], "R": [...], "S": [...]}}`` (storage.py:166-262).

    ``SingularBlock`` is mirrored by ``OracleSingular(step=..., quad=...)``
    (engine.py:320-328).
    """
    m = np.ascontiguousarray(m, dtype=np.float64)
    n = m.shape[0]
    sizes = list(sizes) if sizes is not None else default_sizes(n)
    nb = len(sizes)
    if nb & (nb - 1) or sum(sizes) != n:
        raise ValueError("bad sizes")
    off = offsets_of(sizes)
    k = nb.bit_length() - 1
    counts = counts if counts is not None else EngineCounts()
    minv = np.zeros((n, n))
    tsets = {lv: {"L": [None] * (nb >> lv), "R": [None] * (nb >> lv), "S": [None] * (2 * (nb >> lv))}
             for lv in range(1, k + 1)}

    def spans(level, g):
        first = g << level
        half = 1 << (level - 1)
        return first, first + half, first + 2 * half

    def region(src, cid, r0, r1, c0, c1):
        """engine.py:289-309: a block window of M, or of the T_cid S entry covering it."""
        if src == "matrix":
            return m[off[r0]:off[r1], off[c0]:off[c1]]
        span = 1 << cid
        lo = min(r0, c0)
        qp, rel = divmod(lo, span)
        if rel < span // 2:
            entry, p0 = tsets[cid]["S"][2 * qp], qp * span
        else:
            entry, p0 = tsets[cid]["S"][2 * qp + 1], qp * span + span // 2
        if entry is None:
            raise RuntimeError(f"missing T_{cid} S entry")
        base = off[p0]
        return entry[off[r0] - base:off[r1] - base, off[c0] - base:off[c1] - base]

    def diag(src, cid, stepid):
        for p in range(nb):
            blk = region(src, cid, p, p + 1, p, p + 1)
            counts.inversions += 1
            try:
                inv = _leaf(blk, leaf_inverter)
            except OracleSingular as exc:
                raise OracleSingular(exc.block, exc.path, step=stepid, quad=p) from None
            minv[off[p]:off[p + 1], off[p]:off[p + 1]] = inv

    def arrows(src, cid, lvl):
        for g in range(nb >> lvl):
            first, mid, last = spans(lvl, g)
            sa, sd = sizes[first:mid], sizes[mid:last]
            a = region(src, cid, first, mid, first, mid)
            b = region(src, cid, first, mid, mid, last)
            c = region(src, cid, mid, last, first, mid)
            d = region(src, cid, mid, last, mid, last)
            ainv = minv[off[first]:off[mid], off[first]:off[mid]]
            dinv = minv[off[mid]:off[last], off[mid]:off[last]]
            r = np.empty((off[mid] - off[first], off[last] - off[mid]))
            _fox(ainv, sa, sa, b, sd, r, negate=True)
            l_ = np.empty((off[last] - off[mid], off[mid] - off[first]))
            _fox(dinv, sd, sd, c, sa, l_, negate=True)
            s_d = np.array(a, copy=True)
            _fox(b, sa, sd, l_, sa, s_d, accumulate=True)
            s_a = np.array(d, copy=True)
            _fox(c, sd, sa, r, sd, s_a, accumulate=True)
            t = tsets[lvl]
            t["R"][g], t["L"][g], t["S"][2 * g], t["S"][2 * g + 1] = r, l_, s_d, s_a
            counts.multiplies += 2
            counts.reductions += 2

    def updown(level):
        t = tsets[level]
        for g in range(nb >> level):
            first, mid, last = spans(level, g)
            for down in (True, False):
                panel = t["L"][g] if down else t["R"][g]
                if panel is None:
                    raise RuntimeError(f"missing T_{level} L/R {g}")
                s0, s1, d0, d1 = (first, mid, mid, last) if down else (mid, last, first, mid)
                cols = range(first, mid) if down else range(mid, last)
                for col in cols:
                    src = minv[off[s0]:off[s1], off[col]:off[col + 1]]
                    acc = np.zeros((off[d1] - off[d0], off[col + 1] - off[col]))
                    base = off[s0]
                    for kk in range(s1 - s0):
                        j0, j1 = off[s0 + kk] - base, off[s0 + kk + 1] - base
                        mm_acc(panel[:, j0:j1], src[j0:j1, :], acc)
                    minv[off[d0]:off[d1], off[col]:off[col + 1]] = acc
            counts.multiplies += 2

    last_step = total_steps(nb)
    for stepid in range(1, last_step + 1):
        act = decode_step(loopid_for_step(stepid, nb))
        if act["kind"] == "diag":
            diag("matrix", None, stepid)
        elif act["kind"] == "arrows":
            arrows(act["source"], act["cid"], act["sid"])
        else:
            diag("tset", act["cid"], stepid)
            for level in range(1, act["depth"] + 1):
                updown(level)
        if stop_after_step is not None and stepid >= stop_after_step:
            break
    if return_state:
        return minv, tsets
    return minv


def pivot_a_blocks(m, sizes, leaf_inverter=None) -> np.ndarray:
    """The pivot-A recursion of invertor_by_a (recursive.py:83-123, same six
    products per node, same ascending-k multiply) split at diagonal-block
    boundaries instead of n//2, with the partition's blocks as leaves -- the
    device's BI_SCHEDULE_PIVOT_A.  Leaves use
    ``leaf_inverter`` (default: the pivoted gauss_jordan oracle)."""
    m = np.asarray(m, dtype=np.float64)
    sizes = list(sizes)
    off = offsets_of(sizes)
    inv_leaf = leaf_inverter or gauss_jordan

    def node(x, b0, b1, path):
        if b1 - b0 == 1:
            return inv_leaf(x)  # raises the leaf inverter's singular error
        mid = (b0 + b1) // 2
        p = off[mid] - off[b0]
        q = off[b1] - off[mid]
        a, b, c, d = x[:p, :p], x[:p, p:], x[p:, :p], x[p:, p:]
        ainv = node(a, b0, mid, path + ["A"])
        n_ab = np.empty((p, q))
        multiply(ainv, b, n_ab, negate=True)
        ca = np.empty((q, p))
        multiply(c, ainv, ca)
        s_a = d.copy()
        multiply(c, n_ab, s_a, accumulate=True)
        sinv = node(s_a, mid, b1, path + ["SchurA"])
        out = np.empty((p + q, p + q))
        multiply(n_ab, sinv, out[:p, p:])
        out[:p, :p] = ainv
        multiply(out[:p, p:], ca, out[:p, :p], accumulate=True, negate=True)
        multiply(sinv, ca, out[p:, :p], negate=True)
        out[p:, p:] = sinv
        return out

    return node(m, 0, len(sizes), [])


def flops_pivot_a(sizes) -> dict:
    """Flops of pivot_a_blocks: 6pq(p+q) per node, 2b^3 per leaf (= 2n^3 for
    equal power-of-two partitions)."""
    sizes = list(sizes)
    off = offsets_of(sizes)
    out = {"leaves": sum(2.0 * s**3 for s in sizes), "nodes": 0.0}

    def node(b0, b1):
        if b1 - b0 == 1:
            return
        mid = (b0 + b1) // 2
        p, q = off[mid] - off[b0], off[b1] - off[mid]
        out["nodes"] += 6.0 * p * q * (p + q)
        node(b0, mid)
        node(mid, b1)

    node(0, len(sizes))
    out["total"] = out["leaves"] + out["nodes"]
    return out


def flops_engine(sizes) -> dict:
    """Algorithmic flop count of the step engine for a partition:
    leaves 2*b^3 each, arrows 4 GEMMs per quad, up/down 2 GEMMs per quad per
    pass.  Returns {"leaves", "arrows", "updown", "total"}."""
    sizes = list(sizes)
    nb = len(sizes)
    off = offsets_of(sizes)
    k = nb.bit_length() - 1
    out = {"leaves": 0.0, "arrows": 0.0, "updown": 0.0}
    # every leaf block is inverted once per diag action: step 1 + (nb-1) assemble steps
    out["leaves"] = float(nb) * sum(2.0 * s**3 for s in sizes)
    for stepid in range(1, total_steps(nb) + 1):
        act = decode_step(loopid_for_step(stepid, nb))
        if act["kind"] == "arrows":
            lv = act["sid"]
            for g in range(nb >> lv):
                f, mid, last = g << lv, (g << lv) + (1 << (lv - 1)), (g + 1) << lv
                ha, hd = off[mid] - off[f], off[last] - off[mid]
                out["arrows"] += 2.0 * (ha * ha * hd + hd * hd * ha + ha * hd * ha + hd * ha * hd)
        elif act["kind"] == "assemble":
            for lv in range(1, act["depth"] + 1):
                for g in range(nb >> lv):
                    f, mid, last = g << lv, (g << lv) + (1 << (lv - 1)), (g + 1) << lv
                    ha, hd = off[mid] - off[f], off[last] - off[mid]
                    out["updown"] += 2.0 * (hd * ha * ha + ha * hd * hd)
    out["total"] = out["leaves"] + out["arrows"] + out["updown"]
    return out


# ---------------------------------------------------------------------------
# verification metrics (core.py:405-414 and the north-star Frobenius forms)
# ---------------------------------------------------------------------------


def residual_max(m, x) -> float:
    """core.py:405-414: max |m@x - I|."""
    prod = np.asarray(m) @ np.asarray(x)
    prod[np.diag_indices(prod.shape[0])] -= 1.0
    return float(np.max(np.abs(prod)))


def residual_frob(m, x) -> float:
    """||m@x - I||_F."""
    prod = np.asarray(m) @ np.asarray(x)
    prod[np.diag_indices(prod.shape[0])] -= 1.0
    return float(np.linalg.norm(prod))


def lapack_inverse(m) -> np.ndarray:
    """Stand-in oracle for full-size configs, where the restated reference
    (run_inversion: ~4 min per n = 4096 matrix here, hours at 16384) is too
    slow for a test: the third-party LAPACK inverse (numpy.linalg.inv ->
    getrf/getri, partial pivoting; numpy 2.3 with its bundled OpenBLAS).
    Pinned in tests/test_oracle.py against the reference's own outputs
    (golden engine and Gauss-Jordan inverses) and, the
    reference agrees with LAPACK to ~3e-15 at n <= 4096."""
    return np.linalg.inv(np.asarray(m, dtype=np.float64))


def rel_frob(x, ref) -> float:
    """||x - ref||_F / ||ref||_F."""
    return float(np.linalg.norm(np.asarray(x) - np.asarray(ref)) / np.linalg.norm(ref))
