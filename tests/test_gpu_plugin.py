"""The drop-in at the reference's plugin boundary: the
reference's Schur formula drives the B200 leaf kernel through its own
``invert_sub(block, out)`` protocol (schur.py:16-18, 104-111).

The formula here is the oracle's restatement of the reference's
``invert_via_d`` / ``invert_with_fallback`` (schur.py:142-164, 300-333; pinned
bitwise to reference-generated goldens in tests/test_oracle.py), because the
reference package itself does not travel to the GPU box.  The same call with
the real reference package is run by tools/reference_suite.py (record:
profiles/r02_reference_suite.txt).
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bi():
    import paper_2305_11103_b200 as bi

    return bi


def _plugin(bi):
    """gpu_invert_sub with the oracle's singular-block signal (the reference
    formulas catch their own exception type)."""

    def sub(block, out):
        try:
            bi.gpu_invert_sub(block, out)
        except bi.SingularBlock:
            raise oracle.OracleSingular("A", []) from None

    return sub


def test_reference_via_d_with_gpu_invert_sub(bi):
    from paper_2305_11103_b200.workloads import cfg3

    m, split = cfg3(n=900, split=150, rank=75)  # scaled cfg3: singular A11
    got = np.empty_like(m)
    oracle.invert_via_d(m, split, _plugin(bi), got)  # reference formula, B200 sub-inverter
    ref = np.empty_like(m)
    oracle.invert_via_d(m, split, oracle.gj_sub, ref)  # reference formula, reference GJ oracle
    assert oracle.rel_frob(got, ref) <= 1e-9
    n = m.shape[0]
    assert oracle.residual_frob(m, got) <= n * np.finfo(float).eps * np.linalg.cond(m)


def test_reference_fallback_with_gpu_invert_sub(bi):
    """invert_with_fallback(m, split, out, invert_sub=gpu_invert_sub): the
    rank-deficient A11 makes the device leaf raise, and the reference's own
    fallback order moves on to via_d (test_schur.py:227-232)."""
    from paper_2305_11103_b200.workloads import cfg3

    m, split = cfg3(n=600, split=100, rank=50)
    with pytest.raises(bi.SingularBlock):
        bi.gpu_invert_sub(m[:split, :split], np.empty((split, split)))
    out = np.empty_like(m)
    assert oracle.invert_with_fallback(m, split, out, invert_sub=_plugin(bi)) == "via_d"
    ref = np.empty_like(m)
    oracle.invert_via_d(m, split, oracle.gj_sub, ref)
    assert oracle.rel_frob(out, ref) <= 1e-9


def test_gpu_invert_sub_strided_views(bi):
    """The protocol passes non-contiguous views (schur.py:251, 255 pass
    out[:p, :p]) and the callee writes ``out`` in place."""
    g = np.random.default_rng(7)
    big = g.standard_normal((300, 300)) + 300 * np.eye(300)
    out = np.zeros((400, 400))
    bi.gpu_invert_sub(big[50:250, 100:300], out[10:210, 20:220])
    ref = oracle.gauss_jordan(big[50:250, 100:300])
    assert oracle.rel_frob(out[10:210, 20:220], ref) <= 1e-12
    assert not out[:10].any() and not out[210:].any()
