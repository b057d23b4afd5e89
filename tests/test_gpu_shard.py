"""The native column-sharded level scheduler (shard.py,
bi_engine_create_shard / bi_shard_group_run) on one B200: P ranks mapped to
the same GPU (the exchanges are then device-local peer copies, the schedule
and its event ordering are the multi-GPU ones).

* bitwise equal to the single-device engine for P = 1, 2, 4, 8 on uniform
  and ragged partitions (K never split: test_acceptance.py:146-156 analogue);
* the oracle engine with the pivoted GJ leaf within 1e-12 n (a size the
  oracle finishes in seconds);
* stop_after_step: the slab state after step s equals the single engine's;
* a singular leaf is reported as the single engine's SingularBlock(step, quad);
* the one-process-per-GPU transport (pack -> all-gather -> unpack) over
  gloo with two processes on the GPU: bitwise equal as well.
"""

import numpy as np
import pytest

import oracle
from conftest import well_conditioned

pytestmark = pytest.mark.gpu

CASES = [
    (2, [64] * 8), (4, [64] * 8), (8, [64] * 8), (2, [40, 72, 56, 24, 88, 48, 64, 32]),
    (4, [37, 29, 51, 16, 44, 23, 60, 8]), (8, [32] * 16), (2, [128, 96]), (4, [48] * 16),
]


@pytest.fixture(scope="module")
def bi():
    import paper_2305_11103_b200 as bi

    return bi


@pytest.mark.parametrize("P,sizes", CASES)
def test_group_bitwise_vs_single_engine(bi, P, sizes):
    from paper_2305_11103_b200.shard import run_inversion_group

    n = sum(sizes)
    m = well_conditioned(n, 400 + n + P)
    single = bi.run_inversion(m, sizes=sizes).to_dense()
    got = run_inversion_group(m, sizes, P, devices=[0] * P)
    assert np.array_equal(got, single)


def test_group_vs_oracle_engine(bi):
    from paper_2305_11103_b200.shard import run_inversion_group

    sizes = [24, 40, 16, 32, 8, 48, 24, 40]
    n = sum(sizes)
    m = well_conditioned(n, 991)
    got = run_inversion_group(m, sizes, 4, devices=[0] * 4)
    ref = oracle.run_inversion(m, sizes=sizes, leaf_inverter=oracle.gauss_jordan)
    assert np.max(np.abs(got - ref)) <= 1e-12 * n


@pytest.mark.parametrize("stop", [1, 2, 5, 8, 11, 15])
def test_group_stop_after_step(bi, stop):
    from paper_2305_11103_b200.shard import run_inversion_group

    sizes = [32] * 8  # N_s = 15
    n = sum(sizes)
    m = well_conditioned(n, 73)
    single = bi.run_inversion(m, sizes=sizes, stop_after_step=stop).to_dense()
    got = run_inversion_group(m, sizes, 4, stop_after_step=stop, devices=[0] * 4)
    assert np.array_equal(got, single)


def test_group_singular_leaf_reported_like_single_engine(bi):
    from paper_2305_11103_b200.shard import run_inversion_group

    sizes = [16] * 8
    n = sum(sizes)
    m = well_conditioned(n, 5)
    m[80:96, 80:96] = 0.0  # diagonal block 5 singular at step 1
    with pytest.raises(bi.SingularBlock) as single:
        bi.run_inversion(m, sizes=sizes)
    with pytest.raises(bi.SingularBlock) as sharded:
        run_inversion_group(m, sizes, 4, devices=[0] * 4)
    assert (sharded.value.step, sharded.value.quad) == (single.value.step, single.value.quad) == (1, 5)


def test_run_inversion_workers_takes_native_group(bi, monkeypatch):
    """run_inversion(workers=P) -> the native group path (here P clamps to the
    one visible GPU); the thread-per-GPU path maps ranks onto GPU 0."""
    from paper_2305_11103_b200 import distributed

    sizes = [32] * 8
    n = sum(sizes)
    m = well_conditioned(n, 12)
    out = distributed.run_inversion_local(m, sizes, 2, devices=[0, 0])
    assert np.array_equal(out, bi.run_inversion(m, sizes=sizes).to_dense())


def test_plan_matches_python_scheduler(bi):
    """The native exchange plan equals the host scheduler's (distributed.py):
    one exchange per global-level action, groups of 2^l / (N_b/P) ranks (arrows)
    or the rank's own half of them (up/down passes)."""
    from paper_2305_11103_b200.engine import decode_step, loopid_for_step, total_steps
    from paper_2305_11103_b200.shard import NativeShard

    sizes = [16] * 16
    P = 4
    nb, nbp = len(sizes), len(sizes) // P
    expect = []
    for st in range(1, total_steps(nb) + 1):
        a = decode_step(loopid_for_step(st, nb))
        if a.kind == "arrows_and_schur":
            if (1 << a.sid) > nbp:
                expect.append(("arrows", a.sid))
        elif a.kind == "schur_diag_and_assemble":
            expect += [("updown", lv) for lv in range(1, a.depth + 1) if (1 << lv) > nbp]
    for r in range(P):
        sh = NativeShard(sizes, P, r)
        got = [(x["kind"], x["level"]) for x in sh._x]
        assert got == expect
        for x in sh._x:
            gs = (1 << x["level"]) // nbp  # the quad's ranks; an up/down pass exchanges inside its own half
            in_a = r - r // gs * gs < gs // 2
            assert x["in_a"] == in_a
            if x["kind"] == "updown":
                assert x["gs"] == gs // 2 and x["g0"] == r // (gs // 2) * (gs // 2)
            else:
                assert x["gs"] == gs and x["g0"] == r // gs * gs


def test_library_nccl_transport_single_rank(bi):
    """Transport C (NCCL inside the library, bi_nccl.cu) on one rank: the
    dlopen'ed libnccl, a 1-rank world communicator, bi_engine_run_nccl over
    every segment -- bitwise equal to the single engine.  (Ranks > 1 need
    one GPU each: NCCL refuses two ranks on one device.)"""
    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.shard import LibNccl, NativeShard

    if not _lib.lib().bi_nccl_available():
        pytest.skip("libnccl.so.2 not loadable")
    sizes = [48] * 8
    n = sum(sizes)
    m = well_conditioned(n, 31)
    sh = NativeShard(sizes, 1, 0, staging=True)
    sh.load(m)
    tr = LibNccl(1, 0, lambda raw: raw)
    try:
        tr.attach(sh)
        tr.run(sh)
        assert sh.check() is None
        out = np.empty((n, n))
        sh.write_slab(out)
    finally:
        tr.close()
    assert np.array_equal(out, bi.run_inversion(m, sizes=sizes).to_dense())
