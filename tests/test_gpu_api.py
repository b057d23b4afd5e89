"""GPU parity of the remaining public entry points around the hot path:
assemble_updown (engine.py:460-479), invertor_by_ad (recursive.py:366-449),
invertor_with_fallback (recursive.py:470-496), the bench harness (bench.py)
and the CLI (cli.py), each against the oracle / the reference's golden
outputs.

Tolerances: the reference's max-abs criteria (<= 1e-8 n, test_acceptance.py)
plus relative Frobenius <= 1e-9 (north star) for well-conditioned inputs;
1e-12 relative for single assembly passes (one product per entry).
"""

import importlib

import numpy as np
import pytest

import oracle
from conftest import well_conditioned
from tests_golden_inputs import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bi():
    import paper_2305_11103_b200 as bi

    return bi


def _criteria(m, inv, ref):
    n = m.shape[0]
    assert np.max(np.abs(inv - ref)) <= 1e-8 * n
    assert oracle.residual_max(m, inv) <= 1e-8 * n
    assert oracle.rel_frob(inv, ref) <= 1e-9


def _golden_final_tsets(bi, scheme):
    tsets = {lv: bi.ProvisionalSet(scheme, lv) for lv in (1, 2, 3)}
    for key in GOLDEN.files:
        if key.startswith("step8x8_tset_"):
            lv, kind, idx = key[len("step8x8_tset_"):].split("_")
            tsets[int(lv)]._store(kind, int(idx), GOLDEN[key])
    return tsets


@pytest.mark.parametrize("level", [1, 2, 3])
def test_assemble_updown_rebuilds_the_reference_pass(bi, level):
    """Final reference state of [8]*8: zero the level-`level` off-diagonal
    quadrants, run the pass on the device from the reference's own T-set,
    get the reference's M_inv back (step 15 runs passes 1..3, engine.py:391-394)."""
    scheme = bi.partition_from_sizes([8] * 8)
    final = GOLDEN["step8x8_minv_15"]
    minv = bi.BlockMatrix.from_dense(final.copy(), scheme, role="inverse")
    h = 8 * 2 ** (level - 1)
    for g in range(8 >> level):
        a0, a1, a2 = 2 * g * h, (2 * g + 1) * h, (2 * g + 2) * h
        minv.store.data[a1:a2, a0:a1] = 0.0
        minv.store.data[a0:a1, a1:a2] = 0.0
    c = bi.OpCounters()
    bi.assemble_updown(level, minv, _golden_final_tsets(bi, scheme), counters=c)
    assert c.multiplies == 2 * (8 >> level)
    got = minv.to_dense()
    assert np.max(np.abs(got - final)) <= 1e-12 * np.max(np.abs(final))


def test_assemble_updown_missing_entries(bi):
    scheme = bi.partition_from_sizes([8] * 4)
    minv = bi.BlockMatrix.from_dense(np.eye(32), scheme)
    with pytest.raises(bi.MissingProvisionalData):
        bi.assemble_updown(1, minv, {1: bi.ProvisionalSet(scheme, 1)})


@pytest.mark.parametrize("order", [8, 17, 64])
def test_by_ad_small_vs_reference_golden(bi, order):
    m = well_conditioned(order, 30 + order)
    inv, _ = bi.invertor_by_ad(m)
    _criteria(m, inv, GOLDEN[f"by_ad_{order}"])


@pytest.mark.parametrize("order", [600, 1031])
def test_by_ad_recursion_vs_oracle(bi, order):
    """Orders above the device leaf (256) exercise the Eq. 7 node recursion,
    batched (A, D) / (S_D, S_A) leaf pairs included."""
    m = well_conditioned(order, 70 + order)
    c = bi.OpCounters()
    inv, _ = bi.invertor_by_ad(m, c)
    _criteria(m, inv, oracle.gauss_jordan(m))
    # the reported tallies are the reference recursion's (leaf order 2):
    # 4 products + 2 reductions per node, the scratch law's pooled workspace
    assert c.multiplies == 4 * c.nodes and c.reductions == 2 * c.nodes
    assert c.inversions == 3 * c.nodes + 1  # four sub-inversions per node
    if order == 600:  # the device tree: 600 -> 300 -> leaves of 150: 1 + 4 nodes, 16 leaves
        d = bi.device_tree_counters(600, "by_ad")
        assert (d.nodes, d.multiplies, d.reductions, d.inversions) == (5, 20, 10, 16)


def test_by_ad_singular_leaf_path(bi):
    m = well_conditioned(600, 5)
    m[:150, :150] = 0.0  # A of A is singular
    with pytest.raises(bi.SingularBlock) as ei:
        bi.invertor_by_ad(m)
    assert ei.value.path == ["A", "A"]


@pytest.mark.parametrize("order", [6, 16])
def test_with_fallback_permutation_vs_reference(bi, order):
    inv, _ = bi.invertor_with_fallback(np.eye(order)[::-1].copy())
    assert np.array_equal(inv, GOLDEN[f"fallback_rec_perm{order}"])


def test_with_fallback_large_counter_identity(bi):
    """n = 600 reversal: A (300 x 300) is zero, so the top node falls back to
    pivot B; the inverse of the reversal is itself."""
    p = np.eye(600)[::-1].copy()
    c = bi.OpCounters()
    inv, _ = bi.invertor_with_fallback(p, c)
    assert np.array_equal(inv, p)
    assert c.nodes >= 1


def test_bench_harness_on_device(bi):
    B = importlib.import_module("paper_2305_11103_b200.bench")
    recs = B.bench(["a", "inplace", "ad", "parallel", "oracle"], [32, 64, 96, 128, 160], repeats=3)
    samples = [r for r in recs if r.kind == "sample"]
    assert len(samples) == 5 * 5 * 3 and len([r for r in recs if r.kind == "median"]) == 25
    for r in samples:
        assert r.residual <= B.RESIDUAL_BUDGET * r.order and r.seconds > 0
    fit = B.fit_slope([r for r in samples if r.method == "parallel"], 32, 160)
    assert fit.n_points == 15 and np.isfinite(fit.exponent)
    assert B.records_to_csv(recs).startswith(B.CSV_HEADER)


def test_cli_end_to_end(bi, tmp_path, capsys):
    from paper_2305_11103_b200 import cli

    src, out = tmp_path / "m.bin", tmp_path / "inv.bin"
    assert cli.main(["gen", "--order", "256", "--seed", "3", "--out", str(src), "--binary"]) == 0
    assert cli.main(["invert", "--in", str(src), "--out", str(out), "--binary", "--method", "parallel",
                     "--sizes", "64,64,64,64"]) == 0
    text = capsys.readouterr().out
    assert "method parallel  order 256" in text and "multiplies" in text
    m = bi.load_matrix(src)
    _criteria(m, bi.load_matrix(out), oracle.gauss_jordan(m))
    for method in ("a", "inplace", "ad", "oracle"):
        assert cli.main(["verify", "--in", str(src), "--method", method]) == 0
        assert "OK" in capsys.readouterr().out
    assert cli.main(["verify", "--in", str(src), "--inverse", str(out), "--binary"]) == 0
    # a singular input: exit code 2; the counter-identity with --retry recovers
    sing = tmp_path / "s.txt"
    z = np.ones((8, 8))
    bi.save_matrix(z, sing)
    assert cli.main(["invert", "--in", str(sing), "--method", "oracle"]) == cli.EXIT_SINGULAR
    perm = tmp_path / "p.txt"
    assert cli.main(["gen", "--order", "600", "--kind", "permutation", "--out", str(perm)]) == 0
    assert cli.main(["invert", "--in", str(perm), "--method", "ad", "--retry"]) == 0
    # checkpointed run, then resume; a different input against it -> exit 4
    ck = tmp_path / "ck"
    assert cli.main(["invert", "--in", str(src), "--method", "parallel", "--sizes", "64,64,64,64",
                     "--checkpoint-dir", str(ck), "--binary"]) == 0
    assert cli.main(["resume", "--in", str(src), "--checkpoint-dir", str(ck), "--sizes", "64,64,64,64",
                     "--binary"]) == 0
    other = tmp_path / "o.bin"
    assert cli.main(["gen", "--order", "256", "--seed", "4", "--out", str(other), "--binary"]) == 0
    assert cli.main(["resume", "--in", str(other), "--checkpoint-dir", str(ck), "--sizes", "64,64,64,64",
                     "--binary"]) == cli.EXIT_CHECKPOINT
