"""CPU: the product's host logic and its C ABI, without a GPU.

* the shared library loads and exports every symbol include/blockinv_b200.h
  declares (no compute calls);
* partition / step-schedule host logic equals the reference's (golden);
* compute entry points fail loudly without a device (no CPU fallback);
* the product package never imports the oracle.
"""

import ast
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = np.load(ROOT / "tests" / "golden" / "golden.npz")


@pytest.fixture(scope="module")
def bi():
    from paper_2305_11103_b200 import build_native

    build_native.build()
    import paper_2305_11103_b200 as bi

    return bi


def _header_symbols():
    text = (ROOT / "include" / "blockinv_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bi_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(bi):
    lib = bi.load_library()
    syms = _header_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(lib, s), s
    from paper_2305_11103_b200 import _lib

    assert sorted(n for n, _, _ in _lib.SIGNATURES) == syms
    assert lib.bi_version() == 1


def test_library_is_sm100a_only():
    import subprocess

    from paper_2305_11103_b200 import build_native

    build_native.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(build_native.LIB)],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(build_native.LIB)],
                          capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # FP64 tensor pipe in K1


def test_host_abi_validation_without_device(bi):
    """Argument validation happens before any device work."""
    lib = bi.load_library()
    h = bi._lib._vp()
    sizes = (bi._lib._c_i64 * 3)(4, 4, 4)
    assert lib.bi_engine_create(bi._lib.ctypes.byref(h), 3, sizes, 1) == bi._lib.BI_EDIM
    assert b"power of two" in lib.bi_last_error()
    sizes = (bi._lib._c_i64 * 4)(4, 4, 4, 4)
    assert lib.bi_engine_create(bi._lib.ctypes.byref(h), 4, sizes, 2) == 0
    assert lib.bi_engine_workspace_bytes(h) > 0
    out = (bi._lib.ctypes.c_double * 6)()
    assert lib.bi_engine_counters(h, 1, 7, out) == 0
    assert (out[0], out[1], out[2]) == (20.0, 16.0, 10.0)  # same tallies as the reference engine
    assert lib.bi_engine_destroy(h) == 0
    assert lib.bi_gemm(4, 4, 4, 2, None, 4, 0, None, 4, 0, None, 4, 0, None, 4, 0, 1, None) == bi._lib.BI_EDIM
    assert lib.bi_schur2x2(ord("Q"), 10, 3, None, 10, None, 10, None, 0, None, None) == bi._lib.BI_EDIM
    assert lib.bi_inv_workspace_bytes(3, 512) > 3 * 512 * 512 * 8


@pytest.mark.parametrize("sizes", [[512] * 8, [3, 9, 5, 11], [7]])
def test_engine_pivot_a_schedule_counters(bi, sizes):
    """BI_SCHEDULE_PIVOT_A: one step, invertor_by_a tallies (6 multiplies, 2
    accumulating, per node; every block inverted once) and 2n^3 flops."""
    lib = bi.load_library()
    h = bi._lib._vp()
    arr = (bi._lib._c_i64 * len(sizes))(*sizes)
    assert lib.bi_engine_create_ex(bi._lib.ctypes.byref(h), len(sizes), arr, 3, 1) == 0
    assert lib.bi_engine_workspace_bytes(h) > 0
    out = (bi._lib.ctypes.c_double * 6)()
    assert lib.bi_engine_counters(h, 1, 1, out) == 0
    assert lib.bi_engine_counters(h, 1, 2, out) == bi._lib.BI_EDIM  # one step only
    assert lib.bi_engine_counters(h, 1, 1, out) == 0
    nb, n = len(sizes), sum(sizes)
    assert (out[0], out[1], out[2]) == (6.0 * (nb - 1), float(nb), 2.0 * (nb - 1))
    assert out[3] + out[4] == 3 * 2.0 * n**3  # batch of 3
    assert out[4] == 3 * sum(2.0 * s**3 for s in sizes)
    lib.bi_engine_destroy(h)
    assert lib.bi_engine_create_ex(bi._lib.ctypes.byref(h), len(sizes), arr, 1, 7) == bi._lib.BI_EDIM


def test_engine_counters_match_reference_golden(bi):
    """Native counter tallies == reference OpCounters for every golden case."""
    from test_oracle import ENGINE_CASES

    lib = bi.load_library()
    for name, sizes, order, _ in ENGINE_CASES:
        sizes = sizes or list(bi.make_partition(order).sizes)
        h = bi._lib._vp()
        arr = (bi._lib._c_i64 * len(sizes))(*sizes)
        assert lib.bi_engine_create(bi._lib.ctypes.byref(h), len(sizes), arr, 1) == 0
        out = (bi._lib.ctypes.c_double * 6)()
        assert lib.bi_engine_counters(h, 1, 2 * len(sizes) - 1, out) == 0
        lib.bi_engine_destroy(h)
        assert [int(out[0]), int(out[1]), int(out[2])] == list(GOLDEN[f"engine_{name}_counters"]), name


def test_partition_host_logic_vs_golden(bi):
    sizes = GOLDEN["partition_sizes"]
    pos = 0
    for order in GOLDEN["partition_orders"]:
        s = list(bi.make_partition(int(order)).sizes)
        assert list(sizes[pos:pos + len(s)]) == s
        pos += len(s)
    with pytest.raises(bi.InvalidOrder):
        bi.make_partition(1)
    with pytest.raises(bi.InvalidOrder):
        bi.partition_from_sizes([2, 2, 2])
    sch = bi.partition_from_sizes([5, 9, 7, 11])
    assert sch.offsets == (0, 5, 14, 21, 32) and sch.k == 2


@pytest.mark.parametrize("bs", [1, 2, 4, 8, 16, 32, 64])
def test_schedule_host_logic_vs_golden(bi, bs):
    kinds = {bi.engine.INVERT_DIAGONALS: 0, bi.engine.ARROWS_AND_SCHUR: 1, bi.engine.SCHUR_DIAG_AND_ASSEMBLE: 2}
    for s, row in enumerate(GOLDEN[f"plan_{bs}"], start=1):
        p = bi.step_plan(s, bs)
        width = bs.bit_length()
        assert list(p.loopid) == list(row[:width])
        a = p.action
        got = [kinds[a.kind], 1 if a.source == "tset" else 0, -1 if a.cid is None else a.cid,
               -1 if a.sid is None else a.sid, a.depth]
        assert got == list(row[width:])
    for r in range(1, 17):
        for c in range(1, 17):
            assert bi.updown_iteration_map(r, c) == GOLDEN["updown_16"][r - 1][c - 1]


def test_schedule_errors(bi):
    with pytest.raises(bi.OutOfRange):
        bi.loopid_for_step(16, 8)
    with pytest.raises(bi.OutOfRange):
        bi.loopid_for_step(1, 6)
    for bad in ([0, 1], [2, 2, 0], [1, 1], [], [3, 0, 1], [2, 3, 0], [0], [-1, 0]):
        with pytest.raises(bi.MalformedLoopid):
            bi.decode_step(bad)


def test_no_cpu_fallback(bi):
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    m = np.eye(4) * 2.0
    with pytest.raises(bi.NativeUnavailable):
        bi.run_inversion(m)
    with pytest.raises(bi.NativeUnavailable):
        bi.gauss_jordan_oracle(m)
    with pytest.raises(bi.NativeUnavailable):
        bi.multiply(m, m, np.empty((4, 4)))
    with pytest.raises(bi.NativeUnavailable):
        bi.invert_via_d(bi.diagonal_quad(m, 2), None, np.empty((4, 4)))


def test_argument_errors_before_device(bi):
    with pytest.raises(bi.DimensionMismatch):
        bi.multiply(np.ones((2, 3)), np.ones((2, 3)), np.empty((2, 3)))
    with pytest.raises(bi.DimensionMismatch):
        bi.invert_small(np.eye(5), np.empty((5, 5)))
    with pytest.raises(bi.ScratchTooSmall):
        bi.invertor_inplace_by_a(np.eye(4), row_scratch=np.empty(2))
    with pytest.raises(ValueError):  # storage.py:396-397
        bi.run_inversion(np.eye(4), file_backed=True)
    with pytest.raises(ValueError):
        bi.run_inversion(np.eye(4), checkpoint_dir="/tmp/x", schedule="pivot_a")
    import torch

    if not torch.cuda.is_available():
        with pytest.raises(bi.NativeUnavailable):  # checkpointed runs are device runs too: no CPU fallback
            bi.run_inversion(np.eye(4), checkpoint_dir=str(ROOT / "gpurun_out" / "never_written"))
    with pytest.raises(ValueError):
        bi.run_inversion(np.eye(4), workers=0)
    with pytest.raises(bi.DimensionMismatch):
        bi.invert_via_a(bi.diagonal_quad(np.eye(4), 2), None, np.empty((3, 3)))


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2305_11103_b200"
    for py in pkg.rglob("*.py"):
        tree = ast.parse(py.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert all(not a.name.startswith("oracle") for a in node.names), py
            if isinstance(node, ast.ImportFrom):
                assert not (node.module or "").startswith("oracle"), py


def test_recursive_counters_equal_reference_golden():
    """invertor_by_a / invertor_inplace_by_a / invertor_by_ad report the
    reference recursion's OpCounters (every field, incl. peak_scratch and
    schur_scratch) -- replayed bookkeeping, golden from the reference itself
    (tests/golden/make_counters.py) -- not the device tree's."""
    import json
    from pathlib import Path

    from paper_2305_11103_b200.core import OpCounters
    from paper_2305_11103_b200.recursive import _ref_by_a, _ref_by_ad, _ref_inplace

    gold = json.loads((Path(__file__).parent / "golden" / "counters.json").read_text())
    fields = ("multiplies", "inversions", "reductions", "peak_scratch", "schur_scratch", "nodes")
    for n_s, rec in gold.items():
        n = int(n_s)
        c = OpCounters()
        _ref_by_a(n, c)
        assert {f: getattr(c, f) for f in fields} == rec["by_a"], ("by_a", n)
        c = OpCounters()
        c.alloc(n)
        _ref_inplace(n, c)
        c.release(n)
        assert {f: getattr(c, f) for f in fields} == rec["inplace"], ("inplace", n)
        c = OpCounters()
        _ref_by_ad(n, 0, set(), c)
        assert {f: getattr(c, f) for f in fields} == rec["by_ad"], ("by_ad", n)
    for k in range(2, 7):  # test_acceptance.py:132-143 scratch law
        c = OpCounters()
        _ref_by_ad(2 ** k, 0, set(), c)
        assert c.schur_scratch == 2 ** (k + 1) * (2 ** (k - 1) - 1)
