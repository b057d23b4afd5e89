"""GPU parity of the K1 GEMM and K3 batched pivoted Gauss-Jordan kernels,
called through the C ABI (libblockinv_b200.so), against the CPU oracle /
NumPy float64.

Tolerances (float64 throughout):
  GEMM   ||D - D_ref||_F <= 1e-14 * sqrt(K) * (||A||_F ||B||_F + ||C||_F)
  GJ     relative Frobenius error vs the oracle's pivoted GJ <= 1e-12 on
         well-conditioned blocks; exact on permutations / identity.
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


def _gemm_tol(a, b, c, k):
    scale = np.linalg.norm(a) * np.linalg.norm(b) + (np.linalg.norm(c) if c is not None else 0.0)
    return 1e-14 * np.sqrt(max(k, 1)) * scale + 1e-300


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (7, 5, 3), (128, 128, 16), (129, 131, 17), (300, 257, 513),
                                   (64, 700, 33), (512, 512, 512)])
@pytest.mark.parametrize("negate,accumulate", [(False, False), (True, False), (False, True), (True, True)])
def test_gemm_vs_numpy(bi, m, n, k, negate, accumulate):
    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.core import device_gemm

    g = np.random.default_rng(m * 1000 + n + k)
    a, b, c = g.standard_normal((m, k)), g.standard_normal((k, n)), g.standard_normal((m, n))
    da, db, dd = _lib.to_device(a), _lib.to_device(b), _lib.to_device(c)
    device_gemm(da, db, dd, c=dd if accumulate else None, negate=negate)
    got = dd.cpu().numpy()
    ref = (c if accumulate else 0.0) + (-1.0 if negate else 1.0) * (a @ b)
    assert np.linalg.norm(got - ref) <= _gemm_tol(a, b, c if accumulate else None, k)


@pytest.mark.parametrize("m,n,widths", [(128, 64, [16]), (300, 257, [64, 128, 32, 7]), (129, 70, [16, 16, 16, 16, 16, 16, 16, 1]),
                                         (512, 512, [256, 256]), (77, 33, [48, 0, 32]), (5, 3, [0])])
@pytest.mark.parametrize("negate,accumulate", [(False, False), (True, True)])
def test_gemm_kseg_bitwise(bi, m, n, widths, negate, accumulate):
    """K1P (segments read in place, as from peer GPUs) is bitwise equal to K1
    on the gathered operand, and within the GEMM tolerance of NumPy."""
    import torch

    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.core import device_gemm, device_gemm_kseg

    g = np.random.default_rng(m + n + sum(widths))
    k = sum(widths)
    segs_h = [g.standard_normal((m, w)) for w in widths]
    b, c = g.standard_normal((k, n)), g.standard_normal((m, n))
    segs = [_lib.to_device(x) for x in segs_h]
    db = _lib.to_device(b)
    d1, d2 = _lib.to_device(c), _lib.to_device(c)
    device_gemm_kseg(segs, db, d1, c=d1 if accumulate else None, negate=negate)
    a = np.concatenate(segs_h, axis=1) if k else np.zeros((m, 0))
    device_gemm(_lib.to_device(a) if k else _lib.empty_matrix(m, 0), db, d2, c=d2 if accumulate else None, negate=negate)
    torch.cuda.synchronize()
    got = d1.cpu().numpy()
    assert np.array_equal(got, d2.cpu().numpy())
    ref = (c if accumulate else 0.0) + (-1.0 if negate else 1.0) * (a @ b)
    assert np.linalg.norm(got - ref) <= _gemm_tol(a, b, c if accumulate else None, k)


_KSEG_SCRIPT = """
import numpy as np, torch
from paper_2305_11103_b200 import _lib
from paper_2305_11103_b200.core import device_gemm, device_gemm_kseg
g = np.random.default_rng(3)
for m, n, widths in [(1000, 700, [256, 256, 64, 200]), (128, 64, [16]), (300, 1000, [512, 512, 512, 512, 512, 512, 512, 77])]:
    segs_h = [g.standard_normal((m, w)) for w in widths]
    b = g.standard_normal((sum(widths), n)); c = g.standard_normal((m, n))
    d1, d2 = _lib.to_device(c), _lib.to_device(c)
    db = _lib.to_device(b)
    device_gemm_kseg([_lib.to_device(x) for x in segs_h], db, d1, c=d1, negate=True)
    device_gemm(_lib.to_device(np.concatenate(segs_h, axis=1)), db, d2, c=d2, negate=True)
    torch.cuda.synchronize()
    assert np.array_equal(d1.cpu().numpy(), d2.cpu().numpy()), (m, n, widths)
print("KSEG OK")
"""


@pytest.mark.parametrize("cluster", ["1", "2", "4", "8"])
def test_gemm_kseg_cluster_multicast_bitwise(bi, cluster):
    """Every K1P cluster size (TMA multicast of the A slices across 2/4/8 CTAs;
    1 = no cluster) is bitwise equal to K1 on the gathered operand, including
    cluster padding tiles past N and ragged M/K tails."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, BI_KSEG_CLUSTER=cluster)
    r = subprocess.run([sys.executable, "-c", _KSEG_SCRIPT], env=env, capture_output=True, text=True, timeout=240,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "KSEG OK" in r.stdout, r.stderr[-2000:]


def test_gemm_kseg_unaligned_and_errors(bi):
    """Odd-offset segment views take the 8-byte path; a segment boundary off a
    k-tile is rejected (DimensionMismatch), not silently re-tiled."""
    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.core import device_gemm, device_gemm_kseg
    from paper_2305_11103_b200.errors import DimensionMismatch

    g = np.random.default_rng(9)
    big = _lib.to_device(g.standard_normal((301, 303)))
    segs = [big[1:200, 3:35], big[1:200, 101:150]]
    b = big[5:86, 7:160]
    out, ref = _lib.empty_matrix(199, 153), _lib.empty_matrix(199, 153)
    device_gemm_kseg(segs, b, out)
    import torch

    device_gemm(torch.cat(segs, dim=1).contiguous(), b, ref)
    assert np.array_equal(out.cpu().numpy(), ref.cpu().numpy())
    with pytest.raises(DimensionMismatch):
        device_gemm_kseg([big[:10, :20], big[:10, 20:40]], big[:40, :8], _lib.empty_matrix(10, 8))


def test_gemm_unaligned_views(bi):
    """Odd leading dimensions / odd column offsets take the 8-byte copy path."""
    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.core import device_gemm

    g = np.random.default_rng(5)
    big = _lib.to_device(g.standard_normal((301, 303)))
    a = big[1:200, 3:120]   # odd column offset
    b = big[5:122, 7:160]
    out = _lib.empty_matrix(199, 153)
    device_gemm(a, b, out)
    ref = a.cpu().numpy() @ b.cpu().numpy()
    assert np.linalg.norm(out.cpu().numpy() - ref) <= _gemm_tol(ref, np.eye(1), None, 117) * 10


def test_multiply_numpy_api(bi, rng):
    """core.multiply semantics (core.py:142-170): zero-then-accumulate, negate."""
    a, b = rng.uniform(-1, 1, (9, 6)), rng.uniform(-1, 1, (6, 5))
    out = rng.uniform(-1, 1, (9, 5))
    base = out.copy()
    bi.multiply(a, b, out, accumulate=True, negate=True)
    assert np.max(np.abs(out - (base - a @ b))) <= 1e-14
    bi.multiply(a, b, out)
    assert np.max(np.abs(out - a @ b)) <= 1e-14
    naive = np.zeros((9, 5))
    for i in range(9):
        for j in range(5):
            for kk in range(6):
                naive[i, j] += a[i, kk] * b[kk, j]
    assert np.max(np.abs(out - naive)) <= 1e-14  # test_core.py:55-60


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 17, 31, 32, 33, 64, 100, 255, 256, 257, 512, 513, 1000])
def test_gj_inverse_vs_oracle(bi, n):
    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.core import device_inverse

    count = 3
    ms = np.stack([well_conditioned(n, 100 * n + i) for i in range(count)])
    dm = _lib.to_device(ms)
    dout = _lib.empty_matrix(n, n, batch=count)
    info = device_inverse(dm, dout)
    assert (info == 0).all()
    got = dout.cpu().numpy()
    for i in range(count):
        ref = oracle.gauss_jordan(ms[i])
        assert oracle.rel_frob(got[i], ref) <= 1e-12, (n, i)


@pytest.mark.parametrize("n", [200, 700])
def test_gj_needs_pivoting(bi, n):
    """Zero leading diagonal: only a pivoted elimination survives."""
    g = np.random.default_rng(n)
    m = g.standard_normal((n, n))
    m[0, 0] = 0.0
    m[:, 1] *= 1e-3
    ref = oracle.gauss_jordan(m)
    got = bi.gauss_jordan_oracle(m)
    assert oracle.rel_frob(got, ref) <= 1e-9 * np.linalg.cond(m) * 1e-3 + 1e-10
    assert oracle.residual_frob(m, got) <= 1e-10 * n


def test_gj_exact_cases(bi):
    p = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert np.array_equal(bi.gauss_jordan_oracle(p), p)  # test_core.py:231-233
    for order in (1, 3, 17):
        assert np.array_equal(bi.gauss_jordan_oracle(np.eye(order)), np.eye(order))
    rev = np.eye(40)[::-1].copy()
    assert np.array_equal(bi.gauss_jordan_oracle(rev), rev)


def test_gj_singular(bi):
    with pytest.raises(bi.SingularMatrix):
        bi.gauss_jordan_oracle(np.ones((3, 3)))  # test_core.py:240-242
    with pytest.raises(bi.SingularMatrix):
        bi.gauss_jordan_oracle(np.zeros((5, 5)))
    g = np.random.default_rng(0)
    u, v = g.standard_normal((300, 150)), g.standard_normal((300, 150))
    with pytest.raises(bi.SingularMatrix):
        bi.gauss_jordan_oracle(u @ v.T)  # the cfg3 A11 construction
    with pytest.raises(bi.SingularBlock):
        bi.invert_small(np.ones((2, 2)), np.empty((2, 2)))


def test_invert_small_kats(bi):
    out = np.empty((2, 2))
    bi.invert_small(np.eye(2), out)
    assert np.array_equal(out, np.eye(2))
    bi.invert_small(np.array([[2.0, 0.0], [0.0, 4.0]]), out)
    assert np.array_equal(out, [[0.5, 0.0], [0.0, 0.25]])
    o1 = np.empty((1, 1))
    bi.invert_small(np.array([[5.0]]), o1)
    assert o1[0, 0] == 0.2
    m = np.array([[1.0, 1.0, 2.0, 0.5], [1.0, 1.0, 0.25, 3.0], [2.0, 0.5, 9.0, 0.1], [0.5, 2.0, 0.2, 8.0]])
    o4 = np.empty((4, 4))
    bi.invert_small(m, o4)  # leading 2x2 singular (test_core.py:201-214)
    assert oracle.residual_max(m, o4) <= 1e-10
    with pytest.raises(bi.DimensionMismatch):
        bi.invert_small(np.eye(5), np.empty((5, 5)))


def test_residual_kernel(bi):
    m = well_conditioned(300, 9)
    x = oracle.gauss_jordan(m)
    # rounding-level residuals: agreement to 1e-13 (summation orders differ)
    assert abs(bi.residual_norm(m, x) - oracle.residual_max(m, x)) <= 1e-13
    assert abs(bi.residual_frobenius(m, x) - oracle.residual_frob(m, x)) <= 1e-13
    g = np.random.default_rng(1)
    y = x + 1e-6 * g.standard_normal(x.shape)  # a residual far above rounding must match closely
    assert abs(bi.residual_frobenius(m, y) - oracle.residual_frob(m, y)) <= 1e-10 * oracle.residual_frob(m, y)
    assert bi.residual_norm(np.eye(4), np.eye(4)) == 0.0


def test_inverse_pointer_table_form(bi):
    """bi_inv_batched_ptrs: equal-order blocks scattered over different buffers
    (odd leading dimensions, different source/destination strides) equal the
    oracle's pivoted GJ, and a singular block is flagged in its slot."""
    import torch

    from paper_2305_11103_b200.core import device_inverse_list

    n = 48
    mats = [well_conditioned(n, 300 + i) for i in range(5)]
    mats[3] = np.ones((n, n))  # singular
    bufs = [torch.zeros((n + 7, n + 13), dtype=torch.float64, device="cuda") for _ in range(5)]
    outs_buf = torch.zeros((5 * n + 3, n + 5), dtype=torch.float64, device="cuda")
    blocks, outs = [], []
    for i, m in enumerate(mats):
        v = bufs[i][3:3 + n, 5:5 + n]
        v.copy_(torch.from_numpy(m))
        blocks.append(v)
        outs.append(outs_buf[1 + i * n:1 + (i + 1) * n, 2:2 + n])
    info = device_inverse_list(blocks, outs).cpu().numpy()
    assert info[3] != 0 and all(info[i] == 0 for i in (0, 1, 2, 4))
    for i in (0, 1, 2, 4):
        assert oracle.rel_frob(outs[i].cpu().numpy(), oracle.gauss_jordan(mats[i])) <= 1e-12


def test_gemm_grouped_ragged(bi):
    """bi_gemm_grouped: 6 independent ragged problems (more than the 4 inline
    descriptors: the table goes through the workspace), negate / accumulate
    mixed, one launch; each equals NumPy."""
    import ctypes

    import torch

    from paper_2305_11103_b200 import _lib

    class Desc(ctypes.Structure):
        _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("k", ctypes.c_int64), ("alpha_sign", ctypes.c_int),
                    ("a", ctypes.c_void_p), ("lda", ctypes.c_int64), ("stride_a", ctypes.c_int64),
                    ("b", ctypes.c_void_p), ("ldb", ctypes.c_int64), ("stride_b", ctypes.c_int64),
                    ("cin", ctypes.c_void_p), ("ldc", ctypes.c_int64), ("stride_c", ctypes.c_int64),
                    ("d", ctypes.c_void_p), ("ldd", ctypes.c_int64), ("stride_d", ctypes.c_int64),
                    ("batch", ctypes.c_int)]

    g = np.random.default_rng(11)
    shapes = [(100, 60, 30), (7, 5, 3), (256, 130, 512), (64, 64, 64), (1, 300, 17), (200, 1, 9)]
    keep, descs, refs = [], [], []
    for i, (m, n, k) in enumerate(shapes):
        a, b, c = g.standard_normal((m, k)), g.standard_normal((k, n)), g.standard_normal((m, n))
        da, db, dc = _lib.to_device(a), _lib.to_device(b), _lib.to_device(c)
        neg, acc = i % 2 == 1, i % 3 == 0
        dd = dc if acc else _lib.empty_matrix(m, n)
        keep += [da, db, dc, dd]
        descs.append(Desc(m, n, k, -1 if neg else 1, _lib.ptr(da), _lib.ld(da), 0, _lib.ptr(db), _lib.ld(db), 0,
                          _lib.ptr(dc) if acc else None, _lib.ld(dc) if acc else 0, 0, _lib.ptr(dd), _lib.ld(dd), 0, 1))
        refs.append((dd, (c if acc else 0.0) + (-1.0 if neg else 1.0) * (a @ b), a, b))
    arr = (Desc * len(descs))(*descs)
    L = _lib.lib()
    ws_bytes = L.bi_gemm_grouped_workspace_bytes(len(descs))
    assert ws_bytes > 0
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    rc = L.bi_gemm_grouped(len(descs), ctypes.cast(arr, ctypes.c_void_p), ctypes.c_void_p(ws.data_ptr()), ws_bytes,
                           _lib.stream_ptr())
    assert rc == 0, L.bi_last_error()
    for dd, ref, a, b in refs:
        assert np.linalg.norm(dd.cpu().numpy() - ref) <= _gemm_tol(a, b, ref, a.shape[1]) * 10


def test_init_and_finalize(bi):
    """bi_init / bi_finalize: sm_100 check and setup on a valid
    device, an argument error on an invalid one, and the library keeps
    working after a finalize."""
    import ctypes

    from paper_2305_11103_b200 import _lib

    L = _lib.load_library()
    assert L.bi_init(1, (ctypes.c_int * 1)(0)) == 0
    assert L.bi_init(1, (ctypes.c_int * 1)(4096)) == 2
    assert L.bi_init(0, None) == 2
    assert L.bi_finalize() == 0
    m = well_conditioned(64, 3)
    assert oracle.rel_frob(bi.gauss_jordan_oracle(m), oracle.gauss_jordan(m)) <= 1e-12
