"""Dense FP64 primitives on the B200, behind the reference's signatures
(/root/reference/pkg/src/blockinv/core.py).

NumPy in / NumPy out, as in the reference; every product runs in the K1
DMMA GEMM and every inverse in the K3 pivoted Gauss-Jordan kernel of
libblockinv_b200.so.  There is no CPU compute path.
"""

from __future__ import annotations

from contextlib import contextmanager
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .checkpoint import load_binary, matrix_from_bytes, matrix_to_bytes, save_binary  # noqa: F401 (core API)
from .errors import DimensionMismatch, FormatError, ScratchTooSmall, SingularBlock, SingularMatrix

# Alias checks on every call (core.py:31-47); benchmarks switch them off.
debug_checks = True


@contextmanager
def release_mode():
    """Temporarily disable debug alias checks (core.py:38-47)."""
    global debug_checks
    saved = debug_checks
    debug_checks = False
    try:
        yield
    finally:
        debug_checks = saved


@dataclass
class OpCounters:
    """Block-operation tallies (core.py:61-96)."""

    multiplies: int = 0
    inversions: int = 0
    reductions: int = 0
    peak_scratch: int = 0
    schur_scratch: int = 0
    nodes: int = 0
    _current_scratch: int = field(default=0, repr=False)

    def alloc(self, scalars: int) -> None:
        self._current_scratch += scalars
        if self._current_scratch > self.peak_scratch:
            self.peak_scratch = self._current_scratch

    def release(self, scalars: int) -> None:
        self._current_scratch -= scalars

    def merge(self, other: "OpCounters") -> None:
        self.multiplies += other.multiplies
        self.inversions += other.inversions
        self.reductions += other.reductions
        self.schur_scratch += other.schur_scratch
        self.nodes += other.nodes
        self.peak_scratch = max(self.peak_scratch, other.peak_scratch)


def as_matrix(data) -> np.ndarray:
    """core.py:99-104."""
    m = np.asarray(data, dtype=np.float64)
    if m.ndim != 2:
        raise DimensionMismatch(f"expected a 2-D array, got ndim={m.ndim}")
    return m


def _disjoint(x, y) -> bool:
    return not np.may_share_memory(x, y) or not np.shares_memory(x, y)


# ---------------------------------------------------------------------------
# device-level building blocks (torch tensors in, torch tensors out)
# ---------------------------------------------------------------------------


def device_gemm(a, b, d, c=None, negate=False):
    """K1 on device tensors: d = [c] + (+-1) a @ b.  2-D views with unit
    column stride, or 3-D strided batches ([batch, rows, cols]; a 2-D operand
    is broadcast over the batch); `c` may be `d` (in-place accumulate)."""
    batched = d.dim() == 3
    bsz = d.shape[0] if batched else 1

    def spec(x):
        if x is None:
            return None, 0, 0
        if x.dim() == 3:
            if not batched or x.shape[0] != bsz:
                raise DimensionMismatch(f"gemm batch {tuple(x.shape)} vs {tuple(d.shape)}")
            return _lib.ptr(x), _lib.ld(x), int(x.stride(0))
        return _lib.ptr(x), _lib.ld(x), 0

    m, k = a.shape[-2:]
    n = b.shape[-1]
    if b.shape[-2] != k or tuple(d.shape[-2:]) != (m, n) or (c is not None and tuple(c.shape[-2:]) != (m, n)):
        raise DimensionMismatch(f"gemm {tuple(a.shape)} x {tuple(b.shape)} -> {tuple(d.shape)}")
    (pa, lda, sa), (pb, ldb, sb), (pc, ldc, sc), (pd, ldd, sd) = spec(a), spec(b), spec(c), spec(d)
    rc = _lib.lib().bi_gemm(m, n, k, -1 if negate else 1, pa, lda, sa, pb, ldb, sb, pc, ldc if c is not None else 0,
                            sc, pd, ldd, sd, bsz, _lib.stream_ptr())
    _lib.check(rc, "bi_gemm")


def device_gemm_kseg(segs, b, d, c=None, negate=False):
    """K1P: d = [c] + (+-1) [segs[0] | segs[1] | ...] @ b, reading each 2-D
    segment where it lives (peer GPUs included) instead of gathering it first
    (bi_gemm_kseg).  Every segment but the last must be a multiple of 16
    columns wide; the result is bitwise equal to ``device_gemm`` on the
    concatenation."""
    import ctypes

    m, n = d.shape
    widths = [int(s.shape[1]) for s in segs]
    if any(int(s.shape[0]) != m for s in segs) or b.shape[0] != sum(widths) or b.shape[1] != n \
            or (c is not None and tuple(c.shape) != (m, n)):
        raise DimensionMismatch(f"gemm_kseg {[tuple(s.shape) for s in segs]} x {tuple(b.shape)} -> {tuple(d.shape)}")
    ns = len(segs)
    ptrs = (ctypes.c_void_p * ns)(*[_lib.ptr(s) for s in segs])
    lds = (ctypes.c_int64 * ns)(*[_lib.ld(s) for s in segs])
    ks = (ctypes.c_int64 * ns)(*widths)
    rc = _lib.lib().bi_gemm_kseg(m, n, -1 if negate else 1, ns, ptrs, lds, ks, _lib.ptr(b), _lib.ld(b),
                                 _lib.ptr(c) if c is not None else None, _lib.ld(c) if c is not None else 0,
                                 _lib.ptr(d), _lib.ld(d), _lib.stream_ptr())
    _lib.check(rc, "bi_gemm_kseg")


def device_inverse(blocks, out, sync: bool = True):
    """K3 on a device batch: out[i] = inverse(blocks[i]).  `blocks`/`out` are
    [count, n, n] (or [n, n]) views with unit column stride.  Returns the
    per-block info array (numpy): 0 ok, c+1 first singular pivot column;
    ``sync=False`` returns the device info tensor without waiting."""
    t = _lib.torch()
    single = blocks.dim() == 2
    if single:
        blocks, out = blocks.unsqueeze(0), out.unsqueeze(0)
    count, n, n2 = blocks.shape
    if n != n2 or tuple(out.shape) != (count, n, n):
        raise DimensionMismatch(f"inverse of {tuple(blocks.shape)} into {tuple(out.shape)}")
    L = _lib.lib()
    ws = _lib.workspace(L.bi_inv_workspace_bytes(count, n))
    info = t.zeros((count,), dtype=t.int32, device=blocks.device)
    rc = L.bi_inv_batched(count, n, _lib.ptr(blocks), _lib.ld(blocks), int(blocks.stride(0)),
                          _lib.ptr(out), _lib.ld(out), int(out.stride(0)), _lib.ptr(info),
                          _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    _lib.check(rc, "bi_inv_batched")
    return info.cpu().numpy() if sync else info


def device_inverse_list(blocks, outs):
    """K3 on arbitrary equal-order device blocks: outs[i] = inverse(blocks[i])
    for 2-D views anywhere in device memory (pointer-table form,
    bi_inv_batched_ptrs).  Returns the device info tensor (no host sync)."""
    t = _lib.torch()
    count = len(blocks)
    n = blocks[0].shape[0]
    for b_, o_ in zip(blocks, outs):
        if tuple(b_.shape) != (n, n) or tuple(o_.shape) != (n, n):
            raise DimensionMismatch(f"inverse of {tuple(b_.shape)} into {tuple(o_.shape)} (order {n})")
    dev = blocks[0].device
    # page-locked staging: a pageable H2D copy would block the host until the
    # stream drains, serialising host and device at every call
    tab_h = t.tensor([[b_.data_ptr() for b_ in blocks], [_lib.ld(b_) for b_ in blocks],
                      [o_.data_ptr() for o_ in outs], [_lib.ld(o_) for o_ in outs]], dtype=t.int64).pin_memory()
    tab = tab_h.to(dev, non_blocking=True)
    L = _lib.lib()
    ws = _lib.workspace(L.bi_inv_workspace_bytes(count, n))
    info = t.zeros((count,), dtype=t.int32, device=dev)
    rc = L.bi_inv_batched_ptrs(count, n, _lib.ptr(tab[0]), _lib.ptr(tab[1]), _lib.ptr(tab[2]), _lib.ptr(tab[3]),
                               _lib.ptr(info), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    _lib.check(rc, "bi_inv_batched_ptrs")
    info._bi_keepalive = (tab_h, tab, ws)  # staging and tables live until the caller drops the info
    return info


# ---------------------------------------------------------------------------
# reference-signature entry points (NumPy in / NumPy out)
# ---------------------------------------------------------------------------


# core.py:110-112: the reference dispatches small products to a Python loop
# below this many multiply-adds; on the device every product is K1, so the
# threshold changes nothing (kept for callers that tune it).
_SMALL_PRODUCT = 512
_SMALL_EDGE = 8


def _mm_acc(a, b, out, negate: bool = False) -> None:
    """out += (+-1) a @ b (core.py:115-139): the GEMM primitive every
    product of the reference goes through, here one K1 launch (C = out)."""
    if a.shape[1] != b.shape[0] or out.shape != (a.shape[0], b.shape[1]):
        raise DimensionMismatch(f"_mm_acc {a.shape} x {b.shape} -> {out.shape}")
    if out.size and a.shape[1]:
        dout = _lib.to_device(out)
        device_gemm(_lib.to_device(a), _lib.to_device(b), dout, c=dout, negate=negate)
        _lib.download(dout, out)


def multiply(a, b, out, accumulate=False, negate=False, counters: OpCounters | None = None) -> None:
    """out = (+-1) a @ b, or out += ... when ``accumulate`` (core.py:142-170)."""
    if a.shape[1] != b.shape[0] or out.shape[0] != a.shape[0] or out.shape[1] != b.shape[1]:
        raise DimensionMismatch(f"multiply {a.shape} x {b.shape} -> {out.shape}")
    if debug_checks:
        assert _disjoint(out, a), "out aliases a"
        assert _disjoint(out, b), "out aliases b"
    if out.size:
        da, db = _lib.to_device(a), _lib.to_device(b)
        dout = _lib.to_device(out) if accumulate else _lib.empty_matrix(*out.shape)
        if a.shape[1] == 0:
            if not accumulate:
                out[...] = 0.0
        else:
            device_gemm(da, db, dout, c=dout if accumulate else None, negate=negate)
            _lib.download(dout, out)
    if counters is not None:
        counters.multiplies += 1
        if accumulate:
            counters.reductions += 1


def schur_accumulate(dest, x, y, counters: OpCounters | None = None) -> None:
    """dest += x @ y counted as a reduction only (core.py:173-192)."""
    if x.shape[1] != y.shape[0] or dest.shape != (x.shape[0], y.shape[1]):
        raise DimensionMismatch(f"schur_accumulate {x.shape} x {y.shape} -> {dest.shape}")
    if debug_checks:
        assert _disjoint(dest, x), "dest aliases x"
        assert _disjoint(dest, y), "dest aliases y"
    multiply(x, y, dest, accumulate=True)
    if counters is not None:
        counters.reductions += 1


def multiply_inplace_left(a_inv, target, row_scratch, negate=False, counters=None) -> None:
    """target <- (+-1) a_inv @ target (core.py:195-225).  The scratch contract
    is validated as in the reference; the device product needs none."""
    n = target.shape[0]
    if a_inv.shape != (n, n):
        raise DimensionMismatch(f"inplace left {a_inv.shape} on {target.shape}")
    if row_scratch.shape[0] < n:
        raise ScratchTooSmall(f"need {n} scalars, have {row_scratch.shape[0]}")
    res = np.empty_like(target)
    multiply(np.asarray(a_inv), np.asarray(target), res, negate=negate)
    target[...] = res
    if counters is not None:
        counters.multiplies += 1


def multiply_inplace_right(target, a_inv, row_scratch, negate=False, counters=None) -> None:
    """target <- (+-1) target @ a_inv (core.py:228-253)."""
    n = target.shape[1]
    if a_inv.shape != (n, n):
        raise DimensionMismatch(f"inplace right {target.shape} on {a_inv.shape}")
    if row_scratch.shape[0] < n:
        raise ScratchTooSmall(f"need {n} scalars, have {row_scratch.shape[0]}")
    res = np.empty_like(target)
    multiply(np.asarray(target), np.asarray(a_inv), res, negate=negate)
    target[...] = res
    if counters is not None:
        counters.multiplies += 1


def _invert_host_block(m: np.ndarray) -> tuple[np.ndarray, int]:
    dm = _lib.to_device(m)
    dout = _lib.empty_matrix(*m.shape)
    info = device_inverse(dm, dout)
    return _lib.to_numpy(dout), int(info[0])


def invert_small(m, out, counters: OpCounters | None = None) -> None:
    """Inverse of an order 1-4 block into ``out`` (core.py:350-376) by the K3
    pivoted GJ kernel; singular -> SingularBlock("A")."""
    n = m.shape[0]
    if m.shape != (n, n) or out.shape != (n, n) or not 1 <= n <= 4:
        raise DimensionMismatch(f"invert_small on {m.shape} -> {out.shape}")
    inv, info = _invert_host_block(as_matrix(m))
    if info:
        raise SingularBlock("A", path=[])
    out[...] = inv
    if counters is not None:
        counters.inversions += 1


def gauss_jordan_oracle(m, counters: OpCounters | None = None) -> np.ndarray:
    """Partial-pivot Gauss-Jordan inverse (core.py:379-402) on the device (K3),
    same pivot rule and tolerance 1e-12 * n * max|m|; raises SingularMatrix."""
    m = as_matrix(m)
    n = m.shape[0]
    if m.shape[0] != m.shape[1]:
        raise DimensionMismatch(f"oracle needs a square matrix, got {m.shape}")
    if n == 0:
        return np.zeros((0, 0))
    inv, info = _invert_host_block(m)
    if info:
        raise SingularMatrix(f"no pivot in column {info - 1}")
    if counters is not None:
        counters.inversions += 1
    return np.ascontiguousarray(inv)


def gpu_invert_sub(block, out) -> None:
    """The device leaf inverter in the reference's ``invert_sub(block, out)``
    plugin protocol (schur.py:16-18, 104-111): works on any order, raises
    SingularBlock.  Passing it to the reference's own ``invert_via_d``
    drops the B200 leaf kernel into the reference formula."""
    inv, info = _invert_host_block(as_matrix(block))
    if info:
        raise _caller_singular()("A", path=[])
    out[...] = inv


def _caller_singular():
    """The SingularBlock class of the framework calling the plugin: when the
    reference package (``blockinv``) is the caller, its formulas catch only
    their own SingularBlock (schur.py:104-111, 326-332), so the adapter raises
    that one; otherwise this package's."""
    import sys

    ref = sys.modules.get("blockinv.errors")
    cls = getattr(ref, "SingularBlock", None) if ref is not None else None
    return cls if isinstance(cls, type) and issubclass(cls, Exception) else SingularBlock


def _residual_device(da, dx, batch=False):
    L = _lib.lib()
    t = _lib.torch()
    if not batch:
        da, dx = da.unsqueeze(0), dx.unsqueeze(0)
    z, n, _ = da.shape
    ws = _lib.workspace(L.bi_residual_workspace_bytes(n, z))
    out = t.zeros((2 * z,), dtype=t.float64, device=da.device)
    rc = L.bi_residual(n, z, _lib.ptr(da), _lib.ld(da), int(da.stride(0)),
                       _lib.ptr(dx), _lib.ld(dx), int(dx.stride(0)), _lib.ptr(out),
                       _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    _lib.check(rc, "bi_residual")
    o = out.cpu().numpy().reshape(z, 2)
    return np.sqrt(o[:, 0]), o[:, 1]


def residual_norm(x, x_inv) -> float:
    """max |x @ x_inv - I| (core.py:405-414), computed by K1 + K4 on device."""
    x, x_inv = as_matrix(x), as_matrix(x_inv)
    if x.shape != x_inv.shape or x.shape[0] != x.shape[1]:
        raise DimensionMismatch(f"residual_norm {x.shape} vs {x_inv.shape}")
    _, mx = _residual_device(_lib.to_device(x), _lib.to_device(x_inv))
    return float(mx[0])


def residual_frobenius(x, x_inv) -> float:
    """||x @ x_inv - I||_F (the north-star residual), on device."""
    x, x_inv = as_matrix(x), as_matrix(x_inv)
    if x.shape != x_inv.shape or x.shape[0] != x.shape[1]:
        raise DimensionMismatch(f"residual_frobenius {x.shape} vs {x_inv.shape}")
    fro, _ = _residual_device(_lib.to_device(x), _lib.to_device(x_inv))
    return float(fro[0])


# ---------------------------------------------------------------------------
# matrix files (core.py:415-484): text "rows cols" + rows, or BMAT binary
# (BMAT codec shared with the checkpoint writer, checkpoint.py)
# ---------------------------------------------------------------------------

def _validate_loaded(m: np.ndarray) -> np.ndarray:
    if m.ndim != 2 or m.shape[0] < 1 or m.shape[1] < 1:
        raise FormatError(f"bad matrix shape {m.shape}")
    if not np.all(np.isfinite(m)):
        raise FormatError("matrix contains NaN or Inf entries")
    return np.ascontiguousarray(m, dtype=np.float64)


def save_text(m, path) -> None:
    """core.py:437-442: header line, then one line per row (repr floats)."""
    m = as_matrix(m)
    with open(path, "w") as fh:
        fh.write(f"{m.shape[0]} {m.shape[1]}\n")
        for row in m:
            fh.write(" ".join(repr(float(v)) for v in row) + "\n")


def load_text(path) -> np.ndarray:
    """core.py:445-460."""
    with open(path) as fh:
        header = fh.readline().split()
        if len(header) != 2:
            raise FormatError("first line must be 'rows cols'")
        try:
            rows, cols = int(header[0]), int(header[1])
        except ValueError as exc:
            raise FormatError("non-integer dimensions") from exc
        try:
            data = np.loadtxt(fh, ndmin=2, dtype=np.float64)
        except ValueError as exc:
            raise FormatError(f"bad matrix body: {exc}") from exc
    if data.shape != (rows, cols):
        raise FormatError(f"header says {(rows, cols)}, body is {data.shape}")
    return _validate_loaded(data)


def save_matrix(m, path, binary: bool = False) -> None:
    """core.py:477-478."""
    (save_binary if binary else save_text)(m, path)


def load_matrix(path, binary: bool | None = None) -> np.ndarray:
    """core.py:481-486: sniff the BMAT magic when ``binary`` is None."""
    if binary is None:
        with open(path, "rb") as fh:
            binary = fh.read(4) == b"BMAT"
    return (load_binary if binary else load_text)(path)
