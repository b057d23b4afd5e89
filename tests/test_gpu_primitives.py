"""The reference-signature product primitives on the device against the CPU
oracle: ``fox_block_multiply`` / ``BlockedView``
(engine.py:178-249), ``multiply`` / ``schur_accumulate`` (core.py:142-192) and
``multiply_inplace_left`` / ``multiply_inplace_right`` (core.py:195-253).

All of them are K1 launches behind the reference's call signatures, so each
test compares with the oracle's op-for-op restatement of the reference
(``orc._fox`` / ``mm_acc`` / ``_left_inplace`` / ``_right_inplace``, pinned
bitwise to the reference's golden vectors in tests/test_oracle.py).  K1 sums
in DMMA k-order and the reference in ascending k through NumPy ufuncs, so the
comparison is a forward-error bound, 4 * K * eps * (|a| |b|)_ij per element
(the reference's own check against a naive loop is 1e-14 on O(1) entries,
tests/test_core.py:55-60), and the cases follow the reference's tests: blocked
identity, ragged blocks against the dense product, accumulate with negate,
single-block degenerate, worker-count determinism, shape mismatches, the
scratch contract, counters (tests/test_engine.py:175-245, tests/test_core.py:
43-165).
"""

import numpy as np
import pytest

import oracle
from oracle import blockinv_oracle as orc  # the private restatements (_fox, _left_inplace, ...)

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def bi():
    import paper_2305_11103_b200 as bi

    return bi


def _bound(a, b, extra=None):
    """4 K eps (|a| |b|) (+ |extra|): elementwise forward-error bound of a K-term sum."""
    k = a.shape[1]
    mag = np.abs(a) @ np.abs(b)
    if extra is not None:
        mag = mag + np.abs(extra)
    return 4.0 * max(k, 1) * EPS * mag + 1e-300


def _close(got, ref, bound):
    assert got.shape == ref.shape
    assert np.all(np.abs(got - ref) <= bound), float(np.max(np.abs(got - ref) / bound))


RAGGED = [
    ((24, 40, 16), (32, 8, 56, 24), (48, 16)),      # rows, inner, cols
    ((7,), (5,), (3,)),                               # single block everywhere, tiny (the reference's small path)
    ((64, 64), (64, 64), (64, 64)),
    ((1, 130, 9), (33, 95), (17, 2, 61)),
    ((256,), (128, 128, 64), (200, 56)),
]


@pytest.mark.parametrize("rs,ks,cs", RAGGED)
@pytest.mark.parametrize("negate,accumulate", [(False, False), (True, False), (False, True), (True, True)])
def test_fox_block_multiply_vs_oracle(bi, rng, rs, ks, cs, negate, accumulate):
    a = rng.standard_normal((sum(rs), sum(ks)))
    b = rng.standard_normal((sum(ks), sum(cs)))
    base = rng.standard_normal((sum(rs), sum(cs)))
    got = base.copy()
    c = bi.OpCounters()
    bi.fox_block_multiply(bi.BlockedView(a, rs, ks), bi.BlockedView(b, ks, cs), bi.BlockedView(got, rs, cs),
                          negate=negate, accumulate=accumulate, counters=c)
    ref = base.copy()
    orc._fox(a, list(rs), list(ks), b, list(cs), ref, negate=negate, accumulate=accumulate)
    _close(got, ref, _bound(a, b, base if accumulate else None))
    assert (c.multiplies, c.reductions) == (1, 1 if accumulate else 0)  # engine.py:245-248


def test_fox_blocked_identity_and_worker_determinism(bi, rng):
    """engine.py tests :175-185 (identity blocks reproduce b exactly) and
    :223-235 (the result does not depend on ``workers``)."""
    sizes = (16, 48, 32, 8)
    n = sum(sizes)
    b = rng.standard_normal((n, n))
    out1 = np.empty((n, n))
    bi.fox_block_multiply(bi.BlockedView(np.eye(n), sizes, sizes), bi.BlockedView(b, sizes, sizes),
                          bi.BlockedView(out1, sizes, sizes))
    assert np.array_equal(out1, b)  # 1*x + 0*y terms are exact in any summation order
    a = rng.standard_normal((n, n))
    outs = []
    for workers in (1, 2, 7):
        o = np.empty((n, n))
        bi.fox_block_multiply(bi.BlockedView(a, sizes, sizes), bi.BlockedView(b, sizes, sizes),
                              bi.BlockedView(o, sizes, sizes), workers=workers)
        outs.append(o)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_fox_shape_mismatches(bi, rng):
    """engine.py:186-192, 215-221 / tests/test_engine.py:237-245."""
    a = rng.standard_normal((8, 8))
    with pytest.raises(bi.BlockShapeMismatch):
        bi.BlockedView(a, (4, 3), (4, 4))  # sizes do not cover the data
    av, bv = bi.BlockedView(a, (4, 4), (4, 4)), bi.BlockedView(a.copy(), (2, 6), (4, 4))
    with pytest.raises(bi.BlockShapeMismatch):
        bi.fox_block_multiply(av, bv, bi.BlockedView(np.empty((8, 8)), (4, 4), (4, 4)))  # a cols vs b rows
    with pytest.raises(bi.BlockShapeMismatch):
        bi.fox_block_multiply(av, av, bi.BlockedView(np.empty((8, 8)), (2, 6), (4, 4)))  # out rows vs a rows


@pytest.mark.parametrize("shape", [(5, 7, 3), (64, 64, 64), (129, 33, 257), (1, 300, 1), (300, 1, 300)])
def test_multiply_and_schur_accumulate_vs_oracle(bi, rng, shape):
    m, k, n = shape
    a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
    for negate in (False, True):
        got = np.full((m, n), np.nan)  # multiply overwrites (core.py:165-166)
        bi.multiply(a, b, got, negate=negate)
        ref = np.empty((m, n))
        oracle.multiply(a, b, ref, negate=negate)
        _close(got, ref, _bound(a, b))
    # negate is an exact sign flip of every term (tests/test_core.py:62-72)
    pos, neg = np.empty((m, n)), np.empty((m, n))
    bi.multiply(a, b, pos)
    bi.multiply(a, b, neg, negate=True)
    assert np.array_equal(neg, -pos)
    # schur_accumulate: dest += x @ y, one reduction, no multiply tally (core.py:173-192)
    base = rng.standard_normal((m, n))
    got, ref = base.copy(), base.copy()
    c = bi.OpCounters()
    bi.schur_accumulate(got, a, b, counters=c)
    oracle.mm_acc(a, b, ref)
    _close(got, ref, _bound(a, b, base))
    assert (c.multiplies, c.reductions) == (0, 1)
    with pytest.raises(bi.DimensionMismatch):
        bi.schur_accumulate(np.empty((m + 1, n)), a, b)


def test_multiply_strided_views_and_errors(bi, rng):
    """Operands may be non-contiguous views of a parent (partition.py:37-41);
    the output window is written in place and nothing outside it changes."""
    big = rng.standard_normal((96, 96))
    a, b = big[8:40, 16:80:2], big[0:64:2, 50:90]  # 32 x 32 (strided cols), 32 x 40 (strided rows)
    parent = np.full((64, 64), 7.0)
    out = parent[10:42, 12:52]
    bi.multiply(a, b, out)
    ref = np.empty((32, 40))
    oracle.multiply(np.ascontiguousarray(a), np.ascontiguousarray(b), ref)
    _close(np.ascontiguousarray(out), ref, _bound(a, b))
    mask = np.ones_like(parent, dtype=bool)
    mask[10:42, 12:52] = False
    assert np.all(parent[mask] == 7.0)
    with pytest.raises(bi.DimensionMismatch):
        bi.multiply(a, b[:-1], out)
    with pytest.raises(bi.DimensionMismatch):
        bi.multiply(a, b, np.empty((32, 41)))
    c = bi.OpCounters()
    bi.multiply(a, b, out, counters=c)
    bi.multiply(a, b, out, accumulate=True, counters=c)
    assert (c.multiplies, c.reductions) == (2, 1)  # tests/test_core.py:107-114


@pytest.mark.parametrize("n,w", [(6, 4), (64, 24), (130, 70), (1, 5)])
@pytest.mark.parametrize("negate", [False, True])
def test_multiply_inplace_left_right_vs_oracle(bi, rng, n, w, negate):
    ainv = rng.standard_normal((n, n))
    scratch = np.empty(max(n, w))
    # left: target (n x w) <- (+-) ainv @ target
    t0 = rng.standard_normal((n, w))
    got, ref = t0.copy(), t0.copy()
    c = bi.OpCounters()
    bi.multiply_inplace_left(ainv, got, scratch, negate=negate, counters=c)
    orc._left_inplace(ainv, ref, negate)
    _close(got, ref, _bound(ainv, t0))
    assert c.multiplies == 1
    # right: target (w x n) <- (+-) target @ ainv
    t1 = rng.standard_normal((w, n))
    got, ref = t1.copy(), t1.copy()
    bi.multiply_inplace_right(got, ainv, scratch, negate=negate)
    orc._right_inplace(ref, ainv, negate)
    _close(got, ref, _bound(t1, ainv))


def test_multiply_inplace_contract(bi, rng):
    """Identity leaves the target unchanged; the scratch and shape contracts of
    core.py:206-211, 239-244 are the reference's (ScratchTooSmall,
    DimensionMismatch) although the device product needs no scratch."""
    t = rng.standard_normal((12, 5))
    keep = t.copy()
    bi.multiply_inplace_left(np.eye(12), t, np.empty(12))
    assert np.array_equal(t, keep)
    bi.multiply_inplace_right(t, np.eye(5), np.empty(5))
    assert np.array_equal(t, keep)
    with pytest.raises(bi.ScratchTooSmall):
        bi.multiply_inplace_left(np.eye(12), t, np.empty(11))
    with pytest.raises(bi.ScratchTooSmall):
        bi.multiply_inplace_right(t, np.eye(5), np.empty(4))
    with pytest.raises(bi.DimensionMismatch):
        bi.multiply_inplace_left(np.eye(11), t, np.empty(12))
    with pytest.raises(bi.DimensionMismatch):
        bi.multiply_inplace_right(t, np.eye(6), np.empty(6))
    # a strided target (a column window of a parent) is updated in place
    parent = rng.standard_normal((12, 20))
    win = parent[:, 3:17:2]
    ref = np.ascontiguousarray(win).copy()
    a = rng.standard_normal((12, 12))
    orc._left_inplace(a, ref, False)
    before = parent.copy()
    bi.multiply_inplace_left(a, win, np.empty(12))
    _close(np.ascontiguousarray(parent[:, 3:17:2]), ref, _bound(a, np.ascontiguousarray(before[:, 3:17:2])))
    untouched = np.ones(20, dtype=bool)
    untouched[3:17:2] = False
    assert np.array_equal(parent[:, untouched], before[:, untouched])
