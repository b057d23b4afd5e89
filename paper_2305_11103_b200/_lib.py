"""ctypes binding of libblockinv_b200.so (the C ABI in include/blockinv_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, every compute entry point raises ``NativeUnavailable``.
PyTorch is used only for device memory and the current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import BlockInvError, DimensionMismatch

LIB_PATH = Path(__file__).resolve().parent / "libblockinv_b200.so"

# (name, restype, argtypes) for every symbol the header declares.
_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_vp = ctypes.c_void_p
_pint = ctypes.POINTER(ctypes.c_int)
_pdbl = ctypes.POINTER(ctypes.c_double)

SIGNATURES = [
    ("bi_version", _c_int, []),
    ("bi_last_error", ctypes.c_char_p, []),
    ("bi_init", _c_int, [_c_int, _pint]),
    ("bi_finalize", _c_int, []),
    ("bi_gemm", _c_int, [_c_i64, _c_i64, _c_i64, _c_int,
                         _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64,
                         _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _c_int, _vp]),
    ("bi_gemm_grouped_workspace_bytes", _c_i64, [_c_int]),
    ("bi_gemm_grouped", _c_int, [_c_int, _vp, _vp, _c_i64, _vp]),
    ("bi_gemm_kseg", _c_int, [_c_i64, _c_i64, _c_int, _c_int, _vp, _vp, _vp,
                              _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp]),
    ("bi_inv_workspace_bytes", _c_i64, [_c_int, _c_i64]),
    ("bi_inv_batched", _c_int, [_c_int, _c_i64, _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64,
                                _vp, _vp, _c_i64, _vp]),
    ("bi_inv_batched_ptrs", _c_int, [_c_int, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _vp]),
    ("bi_engine_create", _c_int, [ctypes.POINTER(_vp), _c_int, ctypes.POINTER(_c_i64), _c_int]),
    ("bi_engine_create_ex", _c_int, [ctypes.POINTER(_vp), _c_int, ctypes.POINTER(_c_i64), _c_int, _c_int]),
    ("bi_engine_timeline", _c_int, [_vp, ctypes.POINTER(ctypes.c_float)]),
    ("bi_engine_workspace_bytes", _c_i64, [_vp]),
    ("bi_engine_bind", _c_int, [_vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _vp, _c_i64, _vp]),
    ("bi_engine_run", _c_int, [_vp, _c_int, _c_int, _c_int, _vp]),
    ("bi_engine_run_host", _c_int, [_vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _c_int, _c_int, _c_int,
                                    _vp]),
    ("bi_engine_status", _c_int, [_vp, _pint, _pint, _pint]),
    ("bi_engine_counters", _c_int, [_vp, _c_int, _c_int, _pdbl]),
    ("bi_engine_run_phase", _c_int, [_vp, _c_int, _c_int, _c_int, _vp]),
    ("bi_engine_launches", _c_int, [_vp, _c_int, _c_int, ctypes.POINTER(_c_i64)]),
    ("bi_engine_tset_square", _c_int, [_vp, _c_int, _c_int, _c_int, ctypes.POINTER(_vp),
                                       ctypes.POINTER(_c_i64), ctypes.POINTER(_c_i64)]),
    ("bi_engine_destroy", _c_int, [_vp]),
    ("bi_engine_create_shard", _c_int, [ctypes.POINTER(_vp), _c_int, ctypes.POINTER(_c_i64), _c_int, _c_int,
                                        _c_int]),
    ("bi_engine_shard_info", _c_int, [_vp, ctypes.POINTER(_c_i64)]),
    ("bi_engine_shard_segments", _c_int, [_vp, _c_int, _c_int, _pint, _pint, _pint, _c_int]),
    ("bi_engine_run_ops", _c_int, [_vp, _c_int, _c_int, _c_int, _vp]),
    ("bi_engine_xchg_desc", _c_int, [_vp, _c_int, ctypes.POINTER(_c_i64)]),
    ("bi_engine_shard_buffers", _c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    ("bi_engine_xchg_pack", _c_int, [_vp, _c_int, _vp]),
    ("bi_engine_xchg_unpack", _c_int, [_vp, _c_int, _vp]),
    ("bi_shard_group_run", _c_int, [ctypes.POINTER(_vp), _c_int, ctypes.POINTER(_vp), _c_int, _c_int, _c_int]),
    ("bi_nccl_available", _c_int, []),
    ("bi_nccl_unique_id", _c_int, [ctypes.c_char_p]),
    ("bi_nccl_comm_init", _c_int, [_c_int, ctypes.c_char_p, _c_int, ctypes.POINTER(_vp)]),
    ("bi_nccl_comm_destroy", _c_int, [_vp]),
    ("bi_engine_shard_set_comm", _c_int, [_vp, _vp]),
    ("bi_engine_run_nccl", _c_int, [_vp, _c_int, _c_int, _c_int, _vp]),
    ("bi_schur2x2_workspace_bytes", _c_i64, [_c_i64, _c_i64]),
    ("bi_schur2x2", _c_int, [_c_int, _c_i64, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _pint, _vp]),
    ("bi_inplace_by_a_workspace_bytes", _c_i64, [_c_i64, _c_i64]),
    ("bi_inplace_by_a", _c_int, [_c_i64, _vp, _c_i64, _c_i64, _vp, _c_i64, ctypes.c_char_p, _vp]),
    ("bi_residual_workspace_bytes", _c_i64, [_c_i64, _c_int]),
    ("bi_residual", _c_int, [_c_i64, _c_int, _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64,
                             _vp, _vp, _c_i64, _vp]),
]

BI_OK, BI_ESINGULAR, BI_EDIM, BI_ECUDA, BI_ENCCL, BI_EUNSUPPORTED = range(6)


class NativeUnavailable(BlockInvError, RuntimeError):
    """The CUDA library or a CUDA device is missing (no CPU fallback exists)."""


class NativeError(BlockInvError, RuntimeError):
    """A CUDA/runtime failure reported by the native library."""


class CollectiveError(NativeError):
    """An NCCL failure (or a missing libnccl) in the multi-GPU transport."""


_lib = None


def load_library(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises NativeUnavailable."""
    global _lib
    if _lib is not None:
        return _lib
    # BI_LIB: an alternative build of the same library (A/B timing of kernel variants)
    p = Path(path or os.environ.get("BI_LIB") or LIB_PATH)
    if not p.exists():
        raise NativeUnavailable(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(str(p))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    return load_library()


def check(rc: int, what: str = "") -> int:
    """Map a C-ABI status onto the exception taxonomy (errors.py)."""
    if rc == BI_OK or rc == BI_ESINGULAR:
        return rc
    msg = (lib().bi_last_error() or b"").decode(errors="replace")
    if rc == BI_EDIM:
        raise DimensionMismatch(f"{what}: {msg}")
    if rc == BI_EUNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    if rc == BI_ENCCL:
        raise CollectiveError(f"{what}: {msg}")
    raise NativeError(f"{what}: status {rc}: {msg}")


# ---------------------------------------------------------------------------
# device plumbing (torch for memory and streams only)
# ---------------------------------------------------------------------------

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


_initialised: set = set()


def require_device():
    """Return the current CUDA device; raise NativeUnavailable without one.
    The first use of a device runs ``bi_init`` on it (sm_100 check, kernel
    attributes)."""
    L = load_library()
    t = torch()
    if not t.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible: the B200 library has no CPU fallback")
    dev = t.cuda.current_device()
    if dev not in _initialised:
        ids = (ctypes.c_int * 1)(dev)
        check(L.bi_init(1, ids), "bi_init")
        _initialised.add(dev)
    return t.device("cuda", dev)


def init_devices(devices) -> None:
    """``bi_init`` over several devices: also enables peer access between
    them (the sharded scheduler's slab exchanges over NVLink)."""
    devs = [int(d) for d in devices]
    ids = (ctypes.c_int * len(devs))(*devs)
    check(load_library().bi_init(len(devs), ids), "bi_init")
    _initialised.update(devs)


def stream_ptr() -> int:
    return int(torch().cuda.current_stream().cuda_stream)


def padded_ld(cols: int) -> int:
    """Row pitch in elements: multiple of 4 doubles (32 B) for aligned vector loads."""
    return max(4, (int(cols) + 3) // 4 * 4)


def empty_matrix(rows: int, cols: int, batch: int | None = None):
    """Device float64 matrix (or batch) with padded row pitch; returns the
    [rows, cols] (or [batch, rows, cols]) view of the padded storage."""
    t = torch()
    dev = require_device()
    ld = padded_ld(cols)
    if batch is None:
        return t.empty((rows, ld), dtype=t.float64, device=dev)[:, :cols]
    return t.empty((batch, rows, ld), dtype=t.float64, device=dev)[:, :, :cols]


_STAGE_MIN = 16 << 20  # bytes above which host <-> device copies go through page-locked staging


def to_device(a: np.ndarray):
    """Host float64 matrix (or batch) -> padded device storage.  Large arrays
    are copied into page-locked memory by several threads, then DMA'd (a
    pageable copy runs at one core's speed and blocks the DMA)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 2:
        d = empty_matrix(a.shape[0], a.shape[1])
    else:
        d = empty_matrix(a.shape[1], a.shape[2], batch=a.shape[0])
    t = torch()
    if a.nbytes >= _STAGE_MIN:
        pin = t.empty(a.shape, dtype=t.float64, pin_memory=True)
        _threaded_copy(pin.numpy().reshape(-1, a.shape[-1]), a.reshape(-1, a.shape[-1]))
        d.copy_(pin, non_blocking=True)  # the caching host allocator holds `pin` until this copy has run
        return d
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:  # e.g. a BMAT file's buffer; torch.from_numpy wants a writable array
        a = a.copy()
    d.copy_(t.from_numpy(a))
    return d


_copy_pool = None


def _threaded_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """np.copyto(dst, src) by row chunks on a persistent thread pool (numpy
    drops the GIL in copies): pageable <-> page-locked staging at host-memory
    speed instead of one core's."""
    global _copy_pool
    threads = min(16, os.cpu_count() or 1, max(1, src.nbytes >> 23))
    if threads <= 1 or src.ndim != 2:
        np.copyto(dst, src)
        return
    if _copy_pool is None:
        from concurrent.futures import ThreadPoolExecutor

        _copy_pool = ThreadPoolExecutor(min(16, os.cpu_count() or 1))
    rows = src.shape[0]
    bounds = [rows * i // threads for i in range(threads + 1)]
    list(_copy_pool.map(lambda i: np.copyto(dst[bounds[i]:bounds[i + 1]], src[bounds[i]:bounds[i + 1]]),
                        range(threads)))


def upload(a: np.ndarray):
    """to_device (kept as the name the Schur paths use)."""
    return to_device(a)


def download(d, out: np.ndarray) -> None:
    """out[...] = d (device matrix or batch): large results are DMA'd into
    page-locked memory, then copied into the caller's array by several threads."""
    t = torch()
    if out.nbytes < _STAGE_MIN or out.dtype != np.float64 or out.ndim not in (2, 3):
        out[...] = d.cpu().numpy()
        return
    pin = t.empty(tuple(out.shape), dtype=t.float64, pin_memory=True)
    pin.copy_(d, non_blocking=True)
    t.cuda.current_stream().synchronize()
    if out.ndim == 3 and not out[0].flags.c_contiguous:
        for z in range(out.shape[0]):
            _threaded_copy(out[z], pin[z].numpy())
    else:
        _threaded_copy(out.reshape(-1, out.shape[-1]) if out.flags.c_contiguous else out,
                       pin.numpy().reshape(-1, out.shape[-1]) if out.flags.c_contiguous else pin.numpy())


def to_numpy(d) -> np.ndarray:
    """A new host array with the values of device matrix (or batch) ``d``."""
    out = np.empty(tuple(d.shape), dtype=np.float64)
    download(d, out)
    return out


def workspace(nbytes: int):
    t = torch()
    return t.empty((max(int(nbytes), 256),), dtype=t.uint8, device=require_device())


def ptr(t) -> int:
    return int(t.data_ptr())


def ld(t) -> int:
    return int(t.stride(-2))
