"""CPU: pin the oracle (oracle/, a restatement of the reference) against
(1) golden outputs produced by running the reference itself
    (tests/golden/make_golden.py -> golden.npz), and
(2) the reference test-suite's own known-answer tables.

The oracle is op-for-op the reference, so most comparisons are bitwise.
"""

from pathlib import Path

import numpy as np
import pytest

import oracle
from conftest import well_conditioned

GOLDEN = np.load(Path(__file__).resolve().parent / "golden" / "golden.npz")

# Known-answer tables from the reference tests (test_engine.py:41-69,
# test_partition.py:13-23).
LOOPID_TABLE_B8 = {
    1: [1, 0, 0, 0], 2: [2, 0, 0, 0], 3: [2, 1, 0, 0], 4: [3, 0, 0, 0], 5: [3, 1, 0, 0],
    6: [3, 2, 0, 0], 7: [3, 2, 1, 0], 8: [4, 0, 0, 0], 9: [4, 1, 0, 0], 10: [4, 2, 0, 0],
    11: [4, 2, 1, 0], 12: [4, 3, 0, 0], 13: [4, 3, 1, 0], 14: [4, 3, 2, 0], 15: [4, 3, 2, 1],
}
UPDOWN_MAP_8 = [
    [1, 2, 2, 3, 2, 3, 3, 4], [2, 1, 3, 2, 3, 2, 4, 3], [2, 3, 1, 2, 3, 4, 2, 3], [3, 2, 2, 1, 4, 3, 3, 2],
    [2, 3, 3, 4, 1, 2, 2, 3], [3, 2, 4, 3, 2, 1, 3, 2], [3, 4, 2, 3, 2, 3, 1, 2], [4, 3, 3, 2, 3, 2, 2, 1],
]
TABLE_ROWS = {2: [2], 3: [3], 4: [2, 2], 5: [2, 3], 6: [3, 3], 7: [3, 4], 8: [2, 2, 2, 2], 9: [2, 2, 2, 3],
              21: [2, 2, 2, 3, 3, 3, 3, 3]}

ENGINE_CASES = [
    ("def2", None, 2, 602), ("def3", None, 3, 603), ("def5", None, 5, 605), ("def9", None, 9, 609),
    ("def12", None, 12, 612), ("def21", None, 21, 621), ("def33", None, 33, 633), ("def64", None, 64, 664),
    ("s5_7", [5, 7], 12, 43), ("s3_9_5_11", [3, 9, 5, 11], 28, 44), ("s8x8", [8] * 8, 64, 45),
    ("s16x4", [16] * 4, 64, 46), ("s6x16", [6] * 16, 96, 47),
]


def test_reference_kat_tables():
    for s, row in LOOPID_TABLE_B8.items():
        assert oracle.loopid_for_step(s, 8) == row
    for r in range(1, 9):
        for c in range(1, 9):
            assert oracle.updown_iteration_map(r, c) == UPDOWN_MAP_8[r - 1][c - 1]
    for order, sizes in TABLE_ROWS.items():
        assert oracle.default_sizes(order) == sizes
    assert len(oracle.default_sizes(100)) == 32 and oracle.default_sizes(100) == [3] * 28 + [4] * 4
    assert len(oracle.default_sizes(10000)) == 4096


@pytest.mark.parametrize("bs", [1, 2, 4, 8, 16, 32, 64])
def test_schedule_vs_golden(bs):
    kinds = {"diag": 0, "arrows": 1, "assemble": 2}
    for row in GOLDEN[f"plan_{bs}"]:
        width = bs.bit_length()
        loopid = list(row[:width])
        stepid = sum(1 << (v - 1) for v in loopid if v)
        assert oracle.loopid_for_step(stepid, bs) == loopid
        a = oracle.decode_step(loopid)
        got = [kinds[a["kind"]], 1 if a["source"] == "tset" else 0,
               -1 if a["cid"] is None else a["cid"], -1 if a["sid"] is None else a["sid"], a["depth"]]
        assert got == list(row[width:])


def test_partition_vs_golden():
    sizes = GOLDEN["partition_sizes"]
    pos = 0
    for order in GOLDEN["partition_orders"]:
        s = oracle.default_sizes(int(order))
        assert list(sizes[pos:pos + len(s)]) == s
        pos += len(s)
    assert pos == len(sizes)


@pytest.mark.parametrize("name,sizes,order,seed", ENGINE_CASES)
def test_engine_vs_golden_bitwise(name, sizes, order, seed):
    m = well_conditioned(order, seed)
    c = oracle.EngineCounts()
    got = oracle.run_inversion(m, sizes=sizes, counts=c)
    assert got.tobytes() == GOLDEN[f"engine_{name}"].tobytes()
    assert [c.multiplies, c.inversions, c.reductions] == list(GOLDEN[f"engine_{name}_counters"])


def test_engine_step_state_vs_golden():
    sizes = [8] * 8
    m = well_conditioned(64, 45)
    for step in range(1, 16):
        minv, tsets = oracle.run_inversion(m, sizes=sizes, stop_after_step=step, return_state=True)
        assert minv.tobytes() == GOLDEN[f"step8x8_minv_{step}"].tobytes(), step
    for lv, t in tsets.items():
        for kind in ("L", "R", "S"):
            for idx, arr in enumerate(t[kind]):
                key = f"step8x8_tset_{lv}_{kind}_{idx}"
                assert arr.tobytes() == GOLDEN[key].tobytes(), key


@pytest.mark.parametrize("order", [8, 17, 64])
def test_recursive_and_gj_vs_golden(order):
    m = well_conditioned(order, 30 + order)
    assert oracle.invertor_by_a(m).tobytes() == GOLDEN[f"by_a_{order}"].tobytes()
    x = m.copy()
    oracle.invertor_inplace_by_a(x)
    assert x.tobytes() == GOLDEN[f"inplace_{order}"].tobytes()
    assert oracle.gauss_jordan(m).tobytes() == GOLDEN[f"gj_{order}"].tobytes()
    assert oracle.invertor_by_ad(m).tobytes() == GOLDEN[f"by_ad_{order}"].tobytes()


@pytest.mark.parametrize("sizes", [[32] * 2, [16] * 4, [8] * 8])
def test_pivot_a_blocks_pinned_to_reference_by_a(sizes):
    """Block-level pivot-A (the device's pivot_a schedule) with invertor_by_a
    leaves and equal power-of-two blocks splits exactly where the reference's
    invertor_by_a does (recursive.py:83-123): bitwise equal to the golden
    generated from the reference."""
    m = well_conditioned(64, 94)
    x = oracle.pivot_a_blocks(m, sizes, leaf_inverter=oracle.invertor_by_a)
    assert x.tobytes() == GOLDEN["by_a_64"].tobytes()


@pytest.mark.parametrize("sizes", [[8] * 8, [3, 9, 5, 11], [5, 7], [1], [256] * 16])
def test_pivot_a_flops_are_2n3(sizes):
    n = sum(sizes)
    assert oracle.flops_pivot_a(sizes)["total"] == 2.0 * n**3


def test_formulas_vs_golden():
    m = well_conditioned(60, 3)
    for nm, f in (("a", oracle.invert_via_a), ("d", oracle.invert_via_d), ("ad", oracle.invert_via_ad)):
        out = np.empty((60, 60))
        f(m, 25, oracle.gj_sub, out)
        assert out.tobytes() == GOLDEN[f"via_{nm}_60_25"].tobytes(), nm
    m = well_conditioned(4, 20)
    m[0, 0] = 0.0
    out = np.empty((4, 4))
    assert oracle.invert_with_fallback(m, 1, out) == str(GOLDEN["fallback_kat_name"][0]) == "via_d"
    assert out.tobytes() == GOLDEN["fallback_kat_out"].tobytes()


def test_counterdiagonal_formulas_vs_golden():
    for order, split in ((8, 4), (7, 3)):
        m = well_conditioned(order, 10)
        for nm, f in (("b", oracle.invert_via_b), ("c", oracle.invert_via_c), ("bc", oracle.invert_via_bc)):
            out = np.empty((order, order))
            f(m, split, oracle.small_sub, out)
            assert out.tobytes() == GOLDEN[f"via_{nm}_{order}_{split}"].tobytes(), (nm, order)
    perm2 = np.array([[0.0, 1.0], [1.0, 0.0]])
    out = np.empty((2, 2))
    assert oracle.invert_with_fallback(perm2, 1, out) == str(GOLDEN["fallback_perm2_name"][0]) == "via_b"
    assert np.array_equal(out, GOLDEN["fallback_perm2_out"])


def test_cfg3_shape_vs_golden():
    from tests_golden_inputs import cfg3_small

    m3 = cfg3_small()
    with pytest.raises(oracle.OracleSingularMatrix):
        oracle.gauss_jordan(m3[:20, :20])
    assert GOLDEN["cfg3s_a11_singular"][0] == 1
    out = np.empty_like(m3)
    oracle.invert_via_d(m3, 20, oracle.gj_sub, out)
    assert out.tobytes() == GOLDEN["cfg3s_via_d_gj"].tobytes()


def test_oracle_kats():
    """Reference known-answer tests restated (test_core.py:168-246)."""
    assert np.array_equal(oracle.invert_small(np.eye(2)), np.eye(2))
    assert np.array_equal(oracle.invert_small(np.array([[2.0, 0.0], [0.0, 4.0]])), [[0.5, 0.0], [0.0, 0.25]])
    assert oracle.invert_small(np.array([[5.0]]))[0, 0] == 0.2
    with pytest.raises(oracle.OracleSingular):
        oracle.invert_small(np.zeros((1, 1)))
    with pytest.raises(oracle.OracleSingular):
        oracle.invert_small(np.ones((2, 2)))
    p = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert np.array_equal(oracle.gauss_jordan(p), p)
    with pytest.raises(oracle.OracleSingularMatrix):
        oracle.gauss_jordan(np.ones((3, 3)))
    m = np.array([[1.0, 1.0, 2.0, 0.5], [1.0, 1.0, 0.25, 3.0], [2.0, 0.5, 9.0, 0.1], [0.5, 2.0, 0.2, 8.0]])
    assert oracle.residual_max(m, oracle.invert_small(m)) <= 1e-10
    inv = oracle.run_inversion(np.eye(21))
    assert np.array_equal(inv, np.eye(21))
    with pytest.raises(oracle.OracleSingular) as info:
        oracle.run_inversion(np.eye(4)[::-1].copy())
    assert info.value.step == 1 and info.value.quad is not None


def test_flops_engine_matches_survey():
    """arrows = 2n^3 - 2n^2 b, updown = n^3 - n^2 b, leaves = 2 n^2 b."""
    n, b = 1024, 128
    f = oracle.flops_engine([b] * (n // b))
    assert f["arrows"] == 2 * n**3 - 2 * n**2 * b
    assert f["updown"] == n**3 - n**2 * b
    assert f["leaves"] == 2 * n**2 * b


@pytest.mark.parametrize("name,order,seed", [("s8x8", 64, 45), ("s6x16", 96, 47), ("def64", 64, 664)])
def test_lapack_stand_in_pinned_to_reference(name, order, seed):
    """The full-size stand-in oracle agrees with the reference's own engine
    outputs (golden) far inside the 1e-9 parity bar."""
    m = well_conditioned(order, seed)
    assert oracle.rel_frob(oracle.lapack_inverse(m), GOLDEN[f"engine_{name}"]) <= 1e-13


@pytest.mark.parametrize("order", [8, 17, 64])
def test_lapack_stand_in_vs_reference_gauss_jordan(order):
    m = well_conditioned(order, 30 + order)
    assert oracle.rel_frob(oracle.lapack_inverse(m), GOLDEN[f"gj_{order}"]) <= 1e-13
