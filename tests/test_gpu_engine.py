"""GPU parity of the hot path -- run_inversion (step engine), invert_via_d /
invert_via_a / invert_with_fallback, invertor_inplace_by_a -- against the CPU
oracle (a restatement of the reference, pinned by tests/test_oracle.py).

Tolerances: the reference's own criteria (max|X - X_oracle| <= 1e-8 n and
max|MX - I| <= 1e-8 n, test_acceptance.py:66-77) plus the north star's
relative Frobenius error <= 1e-9 for well-conditioned inputs.
"""

import numpy as np
import pytest

import oracle
from conftest import well_conditioned

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bi():
    import paper_2305_11103_b200 as bi

    return bi


def _assert_ref_criteria(m, inv, ref):
    n = m.shape[0]
    assert np.max(np.abs(inv - ref)) <= 1e-8 * n
    assert oracle.residual_max(m, inv) <= 1e-8 * n
    assert oracle.rel_frob(inv, ref) <= 1e-9


@pytest.mark.parametrize("order", [2, 3, 4, 5, 6, 9, 12, 21, 33, 64, 100])
def test_default_partition_vs_oracle(bi, order):
    m = well_conditioned(order, 600 + order)  # test_engine.py:292-297
    inv = bi.run_inversion(m).to_dense()
    _assert_ref_criteria(m, inv, oracle.gauss_jordan(m))


@pytest.mark.parametrize("sizes", [[5, 7], [8] * 8, [16] * 4, [3, 9, 5, 11], [64] * 8, [37, 64, 1, 90],
                                   [100] * 16, [256, 256], [33] * 32])
def test_explicit_sizes_vs_oracle_engine(bi, sizes):
    n = sum(sizes)
    m = well_conditioned(n, 43 + n)
    inv = bi.run_inversion(m, sizes=sizes).to_dense()
    ref = oracle.run_inversion(m, sizes=sizes, leaf_inverter=oracle.gauss_jordan)
    _assert_ref_criteria(m, inv, ref)


@pytest.mark.parametrize("sizes", [[16] * 8, [7, 9, 12, 4]])
def test_step_state_parity(bi, sizes):
    """M_inv after every step boundary matches the oracle engine's state
    (stop_after_step, engine.py:538-539), and the provisional sets match."""
    n = sum(sizes)
    m = well_conditioned(n, 7 + n)
    nsteps = bi.total_steps(len(sizes))
    for s in range(1, nsteps + 1):
        got = bi.run_inversion(m, sizes=sizes, stop_after_step=s).to_dense()
        ref, tsets = oracle.run_inversion(m, sizes=sizes, stop_after_step=s, leaf_inverter=oracle.gauss_jordan,
                                          return_state=True)
        scale = max(np.abs(ref).max(), 1e-300)
        assert np.max(np.abs(got - ref)) <= 1e-12 * scale * n, s
    # provisional sets after the full run
    from paper_2305_11103_b200.engine import _engine_for

    eng = _engine_for(tuple(sizes), 1)
    off = oracle.offsets_of(sizes)
    for lv, t in tsets.items():
        for g in range(len(sizes) >> lv):
            sq = eng.tset_square(lv, g).cpu().numpy()
            first, mid, last = g << lv, (g << lv) + (1 << (lv - 1)), (g + 1) << lv
            ha = off[mid] - off[first]
            for name, arr, r0, c0 in (("S_D", t["S"][2 * g], 0, 0), ("R", t["R"][g], 0, ha),
                                      ("L", t["L"][g], ha, 0), ("S_A", t["S"][2 * g + 1], ha, ha)):
                win = sq[r0:r0 + arr.shape[0], c0:c0 + arr.shape[1]]
                assert np.max(np.abs(win - arr)) <= 1e-11 * max(np.abs(arr).max(), 1.0), (lv, g, name)


def test_level1_equals_combined_pivot_formula(bi):
    """run_inversion with two blocks is Eq. 7 (test_engine.py:271-277); on the
    device both are the same kernels, so the agreement is to rounding."""
    for order, split in ((5, 2), (6, 3), (7, 3), (300, 140)):
        m = well_conditioned(order, 41 + order)
        sizes = [split, order - split]
        inv = bi.run_inversion(m, sizes=sizes).to_dense()
        direct = np.empty((order, order))
        bi.invert_via_ad(bi.diagonal_quad(m, split), None, direct)
        assert np.max(np.abs(inv - direct)) <= 1e-14 * order


def test_identity_and_singular_reporting(bi):
    inv = bi.run_inversion(np.eye(21)).to_dense()  # test_engine.py:286-290
    assert np.array_equal(inv, np.eye(21))
    p = np.eye(4)[::-1].copy()
    with pytest.raises(bi.SingularBlock) as info:  # test_engine.py:312-317
        bi.run_inversion(p)
    assert info.value.step == 1 and info.value.quad is not None


def test_block_matrix_input_and_scheme_mismatch(bi):
    m = well_conditioned(9, 44)
    bm = bi.BlockMatrix.from_dense(m)
    inv = bi.run_inversion(bm).to_dense()
    assert oracle.residual_max(m, inv) <= 1e-8
    with pytest.raises(bi.SchemeMismatch):
        bi.run_inversion(bm, sizes=[4, 5])


def test_counters(bi):
    c = bi.OpCounters()
    bi.run_inversion(well_conditioned(8, 45), counters=c)
    ref = oracle.EngineCounts()
    oracle.run_inversion(well_conditioned(8, 45), counts=ref)
    assert (c.multiplies, c.inversions, c.reductions) == (ref.multiplies, ref.inversions, ref.reductions)


def test_batch_matches_single(bi):
    sizes = [32] * 8
    ms = np.stack([well_conditioned(256, s) for s in range(3)])
    out = bi.run_inversion_batch(ms, sizes)
    for i in range(3):
        single = bi.run_inversion(ms[i], sizes=sizes).to_dense()
        assert np.array_equal(out[i], single)  # batch lanes are independent and deterministic


def test_deterministic_replay(bi):
    m = well_conditioned(640, 3)
    a = bi.run_inversion(m, sizes=[80] * 8).to_dense()
    b = bi.run_inversion(m, sizes=[80] * 8).to_dense()
    assert a.tobytes() == b.tobytes()


# ---------------------------------------------------------------------------
# config-shaped cases (BASELINE.json configs, scaled where the oracle is slow)
# ---------------------------------------------------------------------------


def test_cfg1_inplace_by_a(bi):
    from paper_2305_11103_b200.workloads import cfg1

    m, sizes = cfg1()
    x = m.copy()
    c = bi.invertor_inplace_by_a(x)
    ref = oracle.gauss_jordan(m)
    _assert_ref_criteria(m, x, ref)
    assert c.multiplies == 6 * c.nodes and c.reductions == 2 * c.nodes
    inv = bi.run_inversion(m, sizes=sizes).to_dense()
    _assert_ref_criteria(m, inv, ref)


def test_cfg3_scaled_via_d_and_fallback(bi):
    """Singular A11 (rank n1/2): via_a must report SingularBlock('A') and the
    fallback must pick via_d (schur.py:300-333, test_schur.py:227-232).  Oracle:
    the reference formula with the reference's pivoted GJ as sub-inverter."""
    from paper_2305_11103_b200.workloads import cfg3

    m, split = cfg3(n=1200, split=200, rank=100)
    ref = np.empty_like(m)
    oracle.invert_via_d(m, split, oracle.gj_sub, ref)
    out = np.empty_like(m)
    bi.invert_via_d(bi.diagonal_quad(m, split), None, out)
    cond = np.linalg.cond(m)
    eps = np.finfo(float).eps
    assert oracle.residual_frob(m, out) <= 10 * m.shape[0] * eps * cond
    assert oracle.rel_frob(out, ref) <= 100 * eps * cond
    with pytest.raises(bi.SingularBlock) as info:
        bi.invert_via_a(bi.diagonal_quad(m, split), None, np.empty_like(m))
    assert info.value.block == "A"
    out2 = np.empty_like(m)
    assert bi.invert_with_fallback(m, split, out2) == "via_d"
    assert np.array_equal(out2, out)


def test_via_formulas_small_kats(bi):
    m = np.zeros((5, 5))
    m[:2, :2] = well_conditioned(2, 1)
    m[2:, 2:] = well_conditioned(3, 2)
    out = np.empty((5, 5))
    bi.invert_via_a(bi.diagonal_quad(m, 2), bi.invert_small, out)  # test_schur.py:30-37
    assert np.max(np.abs(out - oracle.gauss_jordan(m))) <= 1e-12
    assert np.all(out[:2, 2:] == 0.0) and np.all(out[2:, :2] == 0.0)
    out = np.empty((5, 5))
    bi.invert_via_a(bi.diagonal_quad(np.eye(5), 2), bi.invert_small, out)
    assert np.array_equal(out, np.eye(5))
    c = bi.OpCounters()
    out = np.empty((6, 6))
    bi.invert_via_d(bi.diagonal_quad(well_conditioned(6, 7), 3), bi.invert_small, out, c)
    assert (c.multiplies, c.reductions) == (6, 2)
    m = well_conditioned(4, 20)
    m[0, 0] = 0.0
    out = np.empty((4, 4))
    assert bi.invert_with_fallback(m, 1, out) == "via_d"  # test_schur.py:227-232
    assert np.max(np.abs(out - oracle.gauss_jordan(m))) <= 1e-10
    for seed in range(20):  # test_schur.py:71-79
        m = well_conditioned(5, 800 + seed)
        q = bi.diagonal_quad(m, 2)
        oa, od = np.empty((5, 5)), np.empty((5, 5))
        bi.invert_via_a(q, bi.invert_small, oa)
        bi.invert_via_d(q, bi.invert_small, od)
        assert np.max(np.abs(oa - od)) <= 1e-9


def test_reference_style_invert_sub_callable(bi):
    """A foreign Python invert_sub is honoured (plugin protocol)."""
    m = well_conditioned(40, 21)
    calls = []

    def sub(block, out):
        calls.append(block.shape)
        out[...] = oracle.gauss_jordan(block)

    out = np.empty((40, 40))
    assert bi.invert_with_fallback(m, 15, out, invert_sub=sub) == "via_a"
    assert calls == [(15, 15), (25, 25)]
    assert oracle.residual_max(m, out) <= 1e-12


def test_counterdiagonal_formulas(bi):
    """schur.py:167-297 on the device (test_schur.py:95-137, 245-268)."""
    perm2 = np.array([[0.0, 1.0], [1.0, 0.0]])
    for f in (bi.invert_via_b, bi.invert_via_c):
        out = np.empty((2, 2))
        f(bi.counterdiagonal_quad(perm2, 1), bi.invert_small, out)
        assert np.array_equal(out, perm2)
    m = np.zeros((4, 4))
    m[:2, 2:] = well_conditioned(2, 8)
    m[2:, :2] = well_conditioned(2, 9)
    for f in (bi.invert_via_b, bi.invert_via_c, bi.invert_via_bc):
        out = np.empty((4, 4))
        f(bi.counterdiagonal_quad(m, 2), bi.invert_small, out)
        assert oracle.residual_max(m, out) <= 1e-12
    m = well_conditioned(5, 11)
    q = bi.counterdiagonal_quad(m, 2)
    assert q.b.shape == (2, 2) and q.c.shape == (3, 3)
    out = np.empty((5, 5))
    bi.invert_via_b(q, bi.invert_small, out)
    assert oracle.residual_max(m, out) <= 1e-9
    assert bi.invert_with_fallback(perm2, 1, np.empty((2, 2))) == "via_b"
    with pytest.raises(bi.AllPivotsSingular):
        bi.invert_with_fallback(np.zeros((4, 4)), 2, np.empty((4, 4)))
    for seed in range(20):  # all six formulas agree (test_schur.py:245-268)
        m = well_conditioned(6, 3000 + seed)
        outs = []
        for f, mk in ((bi.invert_via_a, bi.diagonal_quad), (bi.invert_via_d, bi.diagonal_quad),
                      (bi.invert_via_b, bi.counterdiagonal_quad), (bi.invert_via_c, bi.counterdiagonal_quad),
                      (bi.invert_via_ad, bi.diagonal_quad), (bi.invert_via_bc, bi.counterdiagonal_quad)):
            out = np.empty((6, 6))
            f(mk(m, 3), bi.invert_small, out)
            outs.append(out)
        for o in outs[1:]:
            assert np.max(np.abs(o - outs[0])) <= 6e-9
    g = np.random.default_rng(5)
    m = g.standard_normal((300, 300)) + 300 * np.eye(300)[::-1]  # counter-diagonal dominant
    ref = oracle.gauss_jordan(m)
    for f in (bi.invert_via_b, bi.invert_via_c, bi.invert_via_bc):
        out = np.empty((300, 300))
        f(bi.counterdiagonal_quad(m, 120), None, out)
        assert oracle.rel_frob(out, ref) <= 1e-12
    ref_b = np.empty((300, 300))
    oracle.invert_via_b(m, 120, oracle.gj_sub, ref_b)
    out = np.empty((300, 300))
    bi.invert_via_b(bi.counterdiagonal_quad(m, 120), None, out)
    assert oracle.rel_frob(out, ref_b) <= 1e-12


def test_cfg3_full_scale_residual(bi):
    """BASELINE config 3 at full size (n=6000, split 1000, rank-500 A11):
    the automatic fallback must take via_d, and the residual must meet the
    north-star bound ||MX - I||_F <= n eps cond(M) (cond ~ 1.1e7 -> 1.5e-5;
    LAPACK itself reaches 1.8e-8)."""
    from paper_2305_11103_b200.workloads import cfg3

    m, split = cfg3()
    out = np.empty_like(m)
    assert bi.invert_with_fallback(m, split, out) == "via_d"
    res = bi.residual_frobenius(m, out)
    assert res <= 6000 * np.finfo(float).eps * 1.1e7, res
    assert res <= 1e-6, res


# --- pivot-A schedule: block-level invertor_by_a recursion ---

@pytest.mark.parametrize("sizes", [[16] * 8, [7, 9, 12, 4], [64] * 8, [37, 64, 1, 90], [256, 256], [33] * 32, [5],
                                   [128] * 4])
def test_pivot_a_schedule_vs_oracle(bi, sizes):
    n = sum(sizes)
    m = well_conditioned(n, 91 + n)
    inv = bi.run_inversion(m, sizes=sizes, schedule="pivot_a").to_dense()
    _assert_ref_criteria(m, inv, oracle.pivot_a_blocks(m, sizes))
    assert oracle.rel_frob(inv, oracle.gauss_jordan(m)) <= 1e-9


def test_pivot_a_batch_lanes_host_io(bi):
    """Batch of 3 (three lanes), page-locked and pageable host buffers, equal
    to the single-matrix runs bitwise; the Eq. 7 engine gives the same inverse
    to 1e-12."""
    import torch

    sizes = [24] * 8
    n = sum(sizes)
    ms = np.stack([well_conditioned(n, 500 + i) for i in range(3)])
    single = np.stack([bi.run_inversion(ms[i], sizes=sizes, schedule="pivot_a").to_dense() for i in range(3)])
    got = bi.run_inversion_batch(ms, sizes, schedule="pivot_a")
    assert np.array_equal(got, single)
    pin_in = torch.from_numpy(ms).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    bi.run_inversion_batch(pin_in.numpy(), sizes, out=pin_out.numpy(), schedule="pivot_a")
    assert np.array_equal(pin_out.numpy(), single)
    eq7 = bi.run_inversion_batch(ms, sizes)
    for i in range(3):
        assert oracle.rel_frob(single[i], eq7[i]) <= 1e-12


def test_pivot_a_singular_leaf_and_arguments(bi):
    sizes = [4] * 4
    m = well_conditioned(16, 3)
    m[:4, :4] = 1.0  # rank-1 leading block: the first leaf of the recursion
    with pytest.raises(bi.SingularBlock) as ei:
        bi.run_inversion(m, sizes=sizes, schedule="pivot_a")
    assert ei.value.step == 1 and ei.value.quad == 0
    with pytest.raises(ValueError):
        bi.run_inversion(well_conditioned(16, 4), sizes=sizes, schedule="pivot_a", stop_after_step=2)
    with pytest.raises(ValueError):
        bi.run_inversion(well_conditioned(16, 4), sizes=sizes, schedule="lu")
    c = bi.OpCounters()
    bi.run_inversion(well_conditioned(16, 4), sizes=sizes, schedule="pivot_a", counters=c)
    assert (c.multiplies, c.inversions, c.reductions) == (18, 4, 6)


# --- edge cases: late singular leaves, batches, NaN, one block, the largest leaf ---

def test_singular_schur_complement_reported_at_its_step(bi):
    """S_D = A - B D^-1 C = 0 in quad 0 of level 1: the leaf inverted at step 3
    (diag from T1) is singular; the device reports the oracle's (step, quad)."""
    m = np.eye(16)
    m[0:4, 4:8] = np.eye(4)
    m[4:8, 0:4] = np.eye(4)
    with pytest.raises(oracle.OracleSingular) as ref:
        oracle.run_inversion(m, sizes=[4] * 4, leaf_inverter=oracle.gauss_jordan)
    with pytest.raises(bi.SingularBlock) as got:
        bi.run_inversion(m, sizes=[4] * 4)
    assert (got.value.step, got.value.quad) == (ref.value.step, ref.value.quad) == (3, 0)


def test_batch_reports_the_singular_matrix(bi):
    ms = np.stack([well_conditioned(64, 70 + i) for i in range(3)])
    ms[1, :8, :8] = 1.0  # rank-1 first leaf of matrix 1
    with pytest.raises(bi.SingularBlock) as got:
        bi.run_inversion_batch(ms, [8] * 8)
    assert got.value.step == 1 and got.value.quad == 0 and got.value.matrix == 1


def test_nan_input_propagates_like_the_reference(bi):
    """NaN ranks as the pivot (numpy.argmax) and never trips the singular
    test (NaN <= tol is false): the result is NaN, no exception, no hang."""
    m = well_conditioned(32, 71)
    m[3, 5] = np.nan
    ref = oracle.run_inversion(m, sizes=[8] * 4, leaf_inverter=oracle.gauss_jordan)
    got = bi.run_inversion(m, sizes=[8] * 4).to_dense()
    assert np.isnan(ref).any() and np.isnan(got).any()


def test_single_block_partition(bi):
    m = well_conditioned(100, 72)
    got = bi.run_inversion(m, sizes=[100]).to_dense()
    _assert_ref_criteria(m, got, oracle.gauss_jordan(m))


def test_largest_leaf_order_8192(bi):
    """K3 at its limit (n = 8192: a 16-CTA cluster per block), checked by the
    device residual (K1 + K4, itself checked against NumPy in test_gpu_kernels)."""
    import torch

    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.core import _residual_device, device_inverse

    n = 8192
    g = torch.Generator(device="cuda")
    g.manual_seed(8192)
    a = torch.randn((1, n, n), generator=g, dtype=torch.float64, device="cuda") / np.sqrt(n)
    a[0].diagonal().add_(2.0)
    x = _lib.empty_matrix(n, n, batch=1)
    info = device_inverse(a, x)
    assert (info == 0).all()
    fro, mx = _residual_device(a, x, batch=True)
    assert fro[0] <= 1e-9 * n and mx[0] <= 1e-10


def test_batch_wider_than_the_lanes(bi):
    """Batch 10 on 8 lanes (two lanes carry two matrices): device-resident and
    page-locked host paths equal the single-matrix runs bitwise."""
    import torch

    sizes = [16] * 8
    ms = np.stack([well_conditioned(128, 80 + i) for i in range(10)])
    single = np.stack([bi.run_inversion(ms[i], sizes=sizes).to_dense() for i in range(10)])
    assert np.array_equal(bi.run_inversion_batch(ms, sizes), single)
    pin_in = torch.from_numpy(ms).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    bi.run_inversion_batch(pin_in.numpy(), sizes, out=pin_out.numpy())
    assert np.array_equal(pin_out.numpy(), single)
    eng = bi.DeviceEngine(sizes, batch=10)
    eng.load(ms)
    eng.run()
    eng.check()
    assert np.array_equal(eng.Minv[:, :, :128].cpu().numpy(), single)


def test_blocks_above_the_k3_limit(bi):
    """Blocks above 8192 (one K3 cluster) invert by the pivot-A recursion with
    K3 leaves (launch_inv_group), in the batched leaf API, the pointer-table
    form, the engine (2 x 9000) and a Schur formula with a 9000 pivot block;
    checked by device residuals, a singular big block reports its column."""
    import torch

    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.core import _residual_device, device_inverse, device_inverse_list

    n = 9000
    g = torch.Generator(device="cuda")
    g.manual_seed(9000)
    a = torch.randn((2, n, n), generator=g, dtype=torch.float64, device="cuda") / np.sqrt(n)
    a[0].diagonal().add_(2.0)
    a[1].diagonal().add_(3.0)
    x = _lib.empty_matrix(n, n, batch=2)
    info = device_inverse(a, x)
    assert (info == 0).all()
    fro, mx = _residual_device(a, x, batch=True)
    assert (fro <= 1e-9 * n).all() and (mx <= 1e-10).all()
    y = torch.empty_like(a[1])
    info2 = device_inverse_list([a[1]], [y]).cpu().numpy()
    assert info2[0] == 0 and torch.equal(y, x[1])
    s = a[0].clone()
    s[5000] = 0.0  # a zero row: singular, found in the recursion's second leaf
    info3 = device_inverse(s, torch.empty_like(s))
    assert info3[0] != 0
    # the engine with two 9000-blocks (n = 18000) and Eq. 3 with a 9000 pivot block
    m = torch.randn((18000, 18000), generator=g, dtype=torch.float64, device="cuda") / np.sqrt(18000.0)
    m.diagonal().add_(2.0)
    mh = m.cpu().numpy()
    inv = bi.run_inversion(mh, sizes=[9000, 9000]).to_dense()
    assert bi.residual_frobenius(mh, inv) <= 1e-9 * 18000
    out = np.empty_like(mh)
    bi.invert_via_d(bi.diagonal_quad(mh, 9000), None, out)
    assert bi.residual_frobenius(mh, out) <= 1e-9 * 18000


@pytest.mark.parametrize("sizes", [[8] * 8, [16] * 8, [3, 9, 5, 11], [24] * 16, [37, 64, 12, 40]])
def test_vs_reference_default_leaf_inverter(bi, sizes):
    """The engine against the oracle engine with the REFERENCE's own default
    leaf inverter -- orders <= 4 analytic, larger blocks by the unpivoted
    invertor_by_a recursion (engine.py:449-457) -- rather than the pivoted GJ
    the device uses: the two leaf algorithms differ only in rounding on these
    well-conditioned inputs, so the inverses agree to the north star's
    relF <= 1e-9."""
    n = sum(sizes)
    m = well_conditioned(n, 77 + n)
    inv = bi.run_inversion(m, sizes=sizes).to_dense()
    ref = oracle.run_inversion(m, sizes=sizes)  # leaf_inverter=None: the reference default
    _assert_ref_criteria(m, inv, ref)
