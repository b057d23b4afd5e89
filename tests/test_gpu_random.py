"""GPU: seeded random sweep over partitions, schedules and entry points
against the oracle (the GPU analogue of the reference's 200-matrix sweep,
test_acceptance.py:45-80): random power-of-two block counts with ragged
block orders 1..200, well-conditioned and non-symmetric normal inputs,
single / batched / pivot-A runs, each with the reference's max-abs criteria
and relF <= 1e-9."""

import numpy as np
import pytest

import oracle
from conftest import well_conditioned

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bi():
    import paper_2305_11103_b200 as bi

    return bi


def _case(seed):
    g = np.random.default_rng(seed)
    nb = int(2 ** g.integers(0, 5))  # 1..16 blocks
    sizes = [int(s) for s in g.integers(1, 201 if nb <= 4 else 61, nb)]
    n = sum(sizes)
    if seed % 2:
        m = well_conditioned(n, seed)
    else:  # N(0,1)/sqrt(n) + 3 I: non-symmetric, cond ~ 2
        m = g.standard_normal((n, n)) / np.sqrt(n) + 3.0 * np.eye(n)
    return m, sizes


def _criteria(m, inv, ref):
    n = m.shape[0]
    assert np.max(np.abs(inv - ref)) <= 1e-8 * n
    assert oracle.residual_max(m, inv) <= 1e-8 * n
    assert oracle.rel_frob(inv, ref) <= 1e-9


@pytest.mark.parametrize("seed", range(24))
def test_random_partition_engine_and_pivot_a(bi, seed):
    m, sizes = _case(seed)
    ref = oracle.gauss_jordan(m)
    _criteria(m, bi.run_inversion(m, sizes=sizes).to_dense(), ref)
    _criteria(m, bi.run_inversion(m, sizes=sizes, schedule="pivot_a").to_dense(), ref)


@pytest.mark.parametrize("seed", range(100, 106))
def test_random_partition_batch(bi, seed):
    m0, sizes = _case(seed)
    n = m0.shape[0]
    g = np.random.default_rng(seed)
    ms = np.stack([m0] + [g.standard_normal((n, n)) / np.sqrt(n) + 3.0 * np.eye(n) for _ in range(2)])
    out = bi.run_inversion_batch(ms, sizes)
    for b in range(ms.shape[0]):
        _criteria(ms[b], out[b], oracle.gauss_jordan(ms[b]))
    assert np.array_equal(out[0], bi.run_inversion(m0, sizes=sizes).to_dense())
