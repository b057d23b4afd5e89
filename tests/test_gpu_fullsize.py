"""GPU parity at the BASELINE configurations' full sizes.

* cfg2 (batch of 4, n = 4096, 8 x 512): every matrix against the LAPACK
  stand-in oracle (pinned to the reference in tests/test_oracle.py):
  relF <= 1e-9 (north star) and the reference's max-abs criteria
  (<= 1e-8 n, test_acceptance.py:66-77); batched and single-matrix public
  entry points bitwise equal; both schedules agree.
* cfg4 (n = 16384, 64 x 256): no CPU oracle fits a test, so the
  size-independent properties: ||A X - I||_F <= n eps cond (cond <~ 10 for
  this generator, measured 4.7 at cfg2), 32 sampled columns checked on the
  host against A x_j = e_j, and the Eq. 7 and pivot-A schedules -- two
  different algorithms -- agreeing to 1e-12.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

EPS = np.finfo(float).eps


@pytest.fixture(scope="module")
def bi():
    import paper_2305_11103_b200 as bi

    return bi


@pytest.fixture(scope="module")
def cfg2_data(bi):
    from paper_2305_11103_b200.workloads import cfg2

    ms, sizes = cfg2(4)
    return ms, sizes, bi.run_inversion_batch(ms, sizes)


def test_cfg2_full_size_vs_lapack(bi, cfg2_data):
    ms, sizes, inv = cfg2_data
    n = ms.shape[1]
    for b in range(ms.shape[0]):
        ref = oracle.lapack_inverse(ms[b])
        assert oracle.rel_frob(inv[b], ref) <= 1e-9
        assert np.max(np.abs(inv[b] - ref)) <= 1e-8 * n
        assert oracle.residual_max(ms[b], inv[b]) <= 1e-8 * n
        assert oracle.residual_frob(ms[b], inv[b]) <= n * EPS * 10.0


def test_cfg2_single_and_batched_bitwise(bi, cfg2_data):
    ms, sizes, inv = cfg2_data
    single = bi.run_inversion(ms[2], sizes=sizes).to_dense()
    assert np.array_equal(single, inv[2])


def test_cfg2_schedules_agree(bi, cfg2_data):
    ms, sizes, inv = cfg2_data
    pa = bi.run_inversion_batch(ms[:2], sizes, schedule="pivot_a")
    for b in range(2):
        assert oracle.rel_frob(pa[b], inv[b]) <= 1e-12


def test_cfg4_full_size_properties(bi):
    from paper_2305_11103_b200.workloads import cfg4

    m, sizes = cfg4()
    n = m.shape[0]
    x = bi.run_inversion(m, sizes=sizes).to_dense()
    res = bi.residual_frobenius(m, x)  # device K1 + K4
    assert res <= n * EPS * 10.0, res
    cols = np.random.default_rng(44).choice(n, 32, replace=False)
    r = m @ x[:, cols]  # host BLAS
    r[cols, np.arange(cols.size)] -= 1.0
    assert np.linalg.norm(r, axis=0).max() <= 1e-12
    xa = bi.run_inversion(m, sizes=sizes, schedule="pivot_a").to_dense()
    assert oracle.rel_frob(xa, x) <= 1e-12
