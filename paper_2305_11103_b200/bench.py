"""Matrix generation, timing sweeps, CSV output and log-log slope fits
(/root/reference/pkg/src/blockinv/bench.py), with every method executed on
the B200.

Same generators, record types, CSV columns and slope fit as the reference, so
a sweep from either implementation can be compared row by row.  Timing wraps
the inversion call only -- NumPy in, NumPy out, so the host<->device copies
are inside the timed region (the reference-facing cost); a warm-up call per
configuration keeps one-time native setup (library load, engine build, graph
capture) out of it.  Residuals are checked on the device (K1 + K4).
"""

from __future__ import annotations

import gc
import math
import time
from dataclasses import dataclass, field

import numpy as np

from .core import OpCounters, gauss_jordan_oracle, release_mode, residual_norm
from .engine import run_inversion
from .errors import InsufficientData, InvalidOrder
from .partition import make_partition
from .recursive import invertor_by_a, invertor_by_ad, invertor_inplace_by_a

KINDS = ("well-conditioned", "permutation", "block-diagonal")
METHODS = ("a", "inplace", "ad", "parallel", "oracle")
RESIDUAL_BUDGET = 1e-8  # per unit of matrix order (bench.py:24)


def _dominant(g: np.random.Generator, order: int) -> np.ndarray:
    """uniform [-1, 1) entries plus 2 * order on the diagonal."""
    blk = g.uniform(-1.0, 1.0, (order, order))
    blk.flat[:: order + 1] += 2.0 * order
    return blk


def generate(order: int, seed: int = 0, kind: str = "well-conditioned") -> np.ndarray:
    """Deterministic test matrices, bit-identical to bench.py:27-61:
    ``well-conditioned`` (one diagonally dominant uniform draw),
    ``permutation`` (the counter-identity, singular diagonal pivots) and
    ``block-diagonal`` (dominant blocks on the default partition, drawn in
    block order from one generator)."""
    if order < 1:
        raise InvalidOrder(f"order must be >= 1, got {order}")
    if kind not in KINDS:
        raise InvalidOrder(f"unknown kind {kind!r}; choose from {KINDS}")
    if kind == "permutation":
        return np.fliplr(np.eye(order)).copy()
    g = np.random.default_rng(seed)
    if kind == "well-conditioned":
        return _dominant(g, order)
    out = np.zeros((order, order))
    if order == 1:  # no partition of order 1
        out[0, 0] = 2.0
        return out
    offs = make_partition(order).offsets
    for lo, hi in zip(offs[:-1], offs[1:]):
        out[lo:hi, lo:hi] = _dominant(g, hi - lo)
    return out


@dataclass
class TimingRecord:
    method: str
    order: int
    workers: int
    seconds: float
    residual: float
    counters: OpCounters = field(default_factory=OpCounters)
    kind: str = "sample"  # "sample" or "median"


@dataclass(frozen=True)
class SlopeFit:
    m_lo: float
    m_hi: float
    exponent: float
    stderr: float
    n_points: int


def _run_method(method: str, m: np.ndarray, workers: int, sizes=None):
    """bench.py:81-97; ``parallel`` is the device step engine
    (``run_inversion``, ``workers`` -> GPU count)."""
    counters = OpCounters()
    if method == "a":
        inv, _ = invertor_by_a(m, counters)
    elif method == "inplace":
        inv = m.copy()
        invertor_inplace_by_a(inv, counters=counters)
    elif method == "ad":
        inv, _ = invertor_by_ad(m, counters)
    elif method == "parallel":
        inv = run_inversion(m, workers=workers, sizes=sizes, counters=counters).to_dense()
    elif method == "oracle":
        inv = gauss_jordan_oracle(m)
        counters = OpCounters()  # the oracle has no block counters
    else:
        raise InvalidOrder(f"unknown method {method!r}")
    return inv, counters


def time_inversion(method: str, m: np.ndarray, workers: int = 1, sizes=None) -> TimingRecord:
    """One timed inversion, alias checks off and the collector paused
    (bench.py:100-116).  ``_run_method`` returns host arrays, so the device
    work has completed when the clock stops."""
    gc_was_on = gc.isenabled()
    gc.disable()
    try:
        with release_mode():
            start = time.perf_counter()
            inv, counters = _run_method(method, m, workers, sizes)
            seconds = time.perf_counter() - start
    finally:
        if gc_was_on:
            gc.enable()
    res = residual_norm(m, inv)
    return TimingRecord(method, m.shape[0], workers, seconds, res, counters)


def bench(methods, orders, workers_list=(1,), repeats: int = 1, seed: int = 0,
          check_residuals: bool = True, warmup: bool = True, sizes_for=None) -> list[TimingRecord]:
    """bench.py:119-158: one record per (method, order, workers, repeat), plus
    the per-configuration median (flagged ``kind="median"``) when
    repeats > 1; a residual above 1e-8 * order fails the sweep.
    ``sizes_for(order)`` optionally gives the engine partition for
    ``parallel`` (default: the reference's default partition)."""
    if repeats < 1:
        raise InvalidOrder(f"repeats must be >= 1, got {repeats}")
    orders = list(orders)
    if orders != sorted(orders):
        raise InvalidOrder("orders must be ascending")
    for method in methods:
        if method not in METHODS:
            raise InvalidOrder(f"unknown method {method!r}")
    records: list[TimingRecord] = []
    for order in orders:
        m = generate(order, seed=seed + order)
        sizes = sizes_for(order) if sizes_for is not None else None
        for method in methods:
            for workers in workers_list:
                if warmup:
                    _run_method(method, m, workers, sizes)
                samples = []
                for _ in range(repeats):
                    rec = time_inversion(method, m, workers, sizes)
                    if check_residuals and rec.residual > RESIDUAL_BUDGET * order:
                        raise ArithmeticError(f"{method} on order {order}: residual {rec.residual:.3e} "
                                              f"exceeds {RESIDUAL_BUDGET * order:.3e}")
                    samples.append(rec)
                records.extend(samples)
                if repeats > 1:
                    mid = sorted(samples, key=lambda r: r.seconds)[len(samples) // 2]
                    records.append(TimingRecord(mid.method, mid.order, mid.workers, mid.seconds, mid.residual,
                                                mid.counters, kind="median"))
    return records


CSV_HEADER = "method,m,workers,seconds,residual,multiplies,inversions,reductions,kind"


def records_to_csv(records) -> str:
    """bench.py:161-171 (same header and column formats)."""
    lines = [CSV_HEADER]
    for r in records:
        lines.append(f"{r.method},{r.order},{r.workers},{r.seconds:.6f},{r.residual!r},"
                     f"{r.counters.multiplies},{r.counters.inversions},{r.counters.reductions},{r.kind}")
    return "\n".join(lines) + "\n"


def write_csv(records, path) -> None:
    with open(path, "w") as fh:
        fh.write(records_to_csv(records))


def fit_slope(records, m_lo: float, m_hi: float) -> SlopeFit:
    """Exponent n of T ~ m**n: ordinary least squares of log T on log m over
    the records with m in [m_lo, m_hi], with the slope's standard error
    (residual variance on n - 2 degrees of freedom) -- bench.py:179-195.
    Fewer than 4 points -> InsufficientData."""
    sel = np.array([(r.order, r.seconds) for r in records if m_lo <= r.order <= m_hi], dtype=np.float64)
    if sel.shape[0] < 4:
        raise InsufficientData(f"{sel.shape[0]} records in [{m_lo}, {m_hi}], need >= 4")
    lx, ly = np.log(sel[:, 0]), np.log(sel[:, 1])
    dx = lx - lx.mean()
    ss = float(dx @ dx)
    slope = float(dx @ (ly - ly.mean())) / ss
    resid = ly - ly.mean() - slope * dx
    dof = sel.shape[0] - 2
    stderr = math.sqrt(max(float(resid @ resid), 0.0) / dof / ss) if dof > 0 else 0.0
    if not math.isfinite(slope):
        raise InsufficientData("slope is not finite")
    return SlopeFit(m_lo, m_hi, slope, stderr, int(sel.shape[0]))
