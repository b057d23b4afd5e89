"""Command-line front end on the B200 (/root/reference/pkg/src/blockinv/cli.py).

Same sub-commands, options, output lines and exit codes as the reference
(0 success, 2 singular pivot or failed verification, 3 I/O / format /
order error, 4 checkpoint mismatch or corruption), so scripts written for
the reference keep working.  Every inversion method runs on the device:
``parallel`` is the native step engine (``--workers`` -> GPU count),
``a`` / ``inplace`` / ``ad`` the device recursions, ``oracle`` the K3
pivoted Gauss-Jordan kernel; residuals are computed by K1 + K4.

    python -m paper_2305_11103_b200 invert --in m.txt --method parallel --sizes 512,512
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from .bench import KINDS, METHODS, RESIDUAL_BUDGET, bench, fit_slope, generate, records_to_csv, write_csv
from .core import OpCounters, gauss_jordan_oracle, load_matrix, residual_norm, save_matrix
from .engine import resolve_workers, run_inversion, total_steps
from .errors import (
    AllPivotsSingular,
    BlockInvError,
    CheckpointCorrupt,
    FormatError,
    InvalidOrder,
    SchemeMismatch,
    SingularBlock,
    SingularMatrix,
)
from .partition import make_partition, partition_from_sizes
from .recursive import invertor_by_a, invertor_by_ad, invertor_inplace_by_a, invertor_with_fallback

EXIT_OK, EXIT_SINGULAR, EXIT_IO, EXIT_CHECKPOINT = 0, 2, 3, 4

# exception class -> exit code, first match wins (cli.py:251-266)
_EXIT_MAP = (
    ((SingularBlock, SingularMatrix, AllPivotsSingular), EXIT_SINGULAR),
    ((CheckpointCorrupt, SchemeMismatch), EXIT_CHECKPOINT),
    ((FormatError, InvalidOrder, OSError), EXIT_IO),
    ((BlockInvError,), EXIT_IO),
)

_RETRYABLE = ("a", "inplace", "ad")


def int_list(text: str) -> list[int]:
    """'a,b,c' -> [a, b, c] (empty items ignored)."""
    return [int(v) for v in text.split(",") if v]


def order_list(text: str) -> list[int]:
    """'a,b,c' or the inclusive range 'lo:hi:step'."""
    if ":" not in text:
        return int_list(text)
    lo, hi, step = map(int, text.split(":"))
    return list(range(lo, hi + 1, step))


def _invert(m: np.ndarray, method: str, workers: int, sizes=None, checkpoint_dir=None, file_backed=False,
            retry=False):
    """Run one method; on a singular pivot of a fixed-pivot recursion and
    with ``retry``, rerun with the per-node pivot fallback (cli.py:63-90)."""
    counters = OpCounters()
    try:
        if method == "parallel":
            inv = run_inversion(m, workers=workers, sizes=sizes, checkpoint_dir=checkpoint_dir,
                                file_backed=file_backed, counters=counters).to_dense()
        elif method == "oracle":
            inv = gauss_jordan_oracle(m, counters)
        elif method == "inplace":
            inv = np.array(m, dtype=np.float64, copy=True)
            invertor_inplace_by_a(inv, counters=counters)
        else:
            inv, _ = {"a": invertor_by_a, "ad": invertor_by_ad}[method](m, counters)
    except SingularBlock:
        if not (retry and method in _RETRYABLE):
            raise
        counters = OpCounters()
        inv, _ = invertor_with_fallback(m, counters)
    return inv, counters


def _load(args, path):
    return load_matrix(path, binary=True if args.binary else None)


def _gen(args) -> int:
    m = generate(args.order, seed=args.seed, kind=args.kind)
    save_matrix(m, args.out, binary=args.binary)
    print(f"wrote {args.kind} matrix of order {args.order} to {args.out}")
    return EXIT_OK


def _partition(args) -> int:
    scheme = partition_from_sizes(args.sizes) if args.sizes else make_partition(args.order)
    print(f"order {scheme.m_n}: N_k = {scheme.n_blocks} diagonal blocks, {total_steps(scheme.n_blocks)} steps")
    print("sizes " + " ".join(map(str, scheme.sizes)))
    return EXIT_OK


def _invert_cmd(args) -> int:
    m = _load(args, args.infile)
    workers = resolve_workers(args.workers)
    inv, c = _invert(m, args.method, workers, args.sizes, args.checkpoint_dir, args.file_backed, args.retry)
    res = residual_norm(m, inv)
    if args.out:
        save_matrix(inv, args.out, binary=args.binary)
    print(f"method {args.method}  order {m.shape[0]}  workers {workers}")
    print(f"residual {res:.3e}")
    print(f"multiplies {c.multiplies}  inversions {c.inversions}  reductions {c.reductions}  "
          f"peak_scratch {c.peak_scratch}")
    return EXIT_OK


def _verify(args) -> int:
    m = _load(args, args.infile)
    if args.inverse:
        print(f"residual {residual_norm(m, _load(args, args.inverse)):.3e}")
        return EXIT_OK
    inv, _ = _invert(m, args.method, resolve_workers(args.workers), args.sizes)
    res = residual_norm(m, inv)
    diff = float(np.max(np.abs(inv - gauss_jordan_oracle(m))))
    budget = RESIDUAL_BUDGET * m.shape[0]
    print(f"method {args.method}  residual {res:.3e}  max|diff vs oracle| {diff:.3e}")
    if max(res, diff) > budget:
        print(f"FAIL: exceeds budget {budget:.3e}")
        return EXIT_SINGULAR
    print("OK")
    return EXIT_OK


def _bench_cmd(args) -> int:
    methods = args.methods.split(",")
    records = bench(methods, order_list(args.orders), workers_list=int_list(args.workers),
                           repeats=args.repeats, seed=args.seed)
    if args.csv:
        write_csv(records, args.csv)
        print(f"wrote {len(records)} rows to {args.csv}")
    else:
        sys.stdout.write(records_to_csv(records))
    if args.fit:
        lo, hi = map(float, args.fit.split(":"))
        for method in methods:
            fit = fit_slope([r for r in records if r.method == method and r.kind == "sample"], lo, hi)
            print(f"{method}: T ~ m^n with n = {fit.exponent:.3f} +- {fit.stderr:.3f} "
                  f"({fit.n_points} points, m in [{lo:g}, {hi:g}])")
    return EXIT_OK


def _resume(args) -> int:
    m = _load(args, args.infile)
    inv = run_inversion(m, workers=resolve_workers(args.workers), sizes=args.sizes,
                        checkpoint_dir=args.checkpoint_dir, file_backed=args.file_backed).to_dense()
    if args.out:
        save_matrix(inv, args.out, binary=args.binary)
    print(f"resumed run complete; residual {residual_norm(m, inv):.3e}")
    return EXIT_OK


_METHOD = dict(choices=METHODS, default="parallel")
# (name, help, handler, [(flags, kwargs), ...]) -- the reference's sub-commands (cli.py:194-248)
_COMMANDS = (
    ("gen", "generate a test matrix", _gen, [
        (("--order",), dict(type=int, required=True)),
        (("--seed",), dict(type=int, default=0)),
        (("--kind",), dict(choices=KINDS, default="well-conditioned")),
        (("--out",), dict(required=True)),
        (("--binary",), dict(action="store_true"))]),
    ("partition", "show the diagonal blocking of an order", _partition, [
        (("order",), dict(type=int)),
        (("--sizes",), dict(type=int_list, default=None))]),
    ("invert", "invert a matrix file", _invert_cmd, [
        (("--in",), dict(dest="infile", required=True)),
        (("--out",), dict(default=None)),
        (("--method",), _METHOD),
        (("--workers",), dict(type=int, default=None)),
        (("--sizes",), dict(type=int_list, default=None)),
        (("--checkpoint-dir",), dict(default=None)),
        (("--file-backed",), dict(action="store_true")),
        (("--retry",), dict(action="store_true", help="on a singular pivot, retry with per-node pivot fallback")),
        (("--binary",), dict(action="store_true"))]),
    ("verify", "check an inversion against the oracle", _verify, [
        (("--in",), dict(dest="infile", required=True)),
        (("--inverse",), dict(default=None, help="verify this inverse file instead")),
        (("--method",), _METHOD),
        (("--workers",), dict(type=int, default=None)),
        (("--sizes",), dict(type=int_list, default=None)),
        (("--binary",), dict(action="store_true"))]),
    ("bench", "timing sweep with CSV output", _bench_cmd, [
        (("--methods",), dict(default="a,inplace,ad")),
        (("--orders",), dict(required=True, help="'a,b,c' or 'lo:hi:step'")),
        (("--workers",), dict(default="1")),
        (("--repeats",), dict(type=int, default=1)),
        (("--seed",), dict(type=int, default=0)),
        (("--csv",), dict(default=None)),
        (("--fit",), dict(default=None, help="'lo:hi' slope-fit range"))]),
    ("resume", "continue a checkpointed run to completion", _resume, [
        (("--in",), dict(dest="infile", required=True)),
        (("--checkpoint-dir",), dict(required=True)),
        (("--out",), dict(default=None)),
        (("--workers",), dict(type=int, default=None)),
        (("--sizes",), dict(type=int_list, default=None)),
        (("--file-backed",), dict(action="store_true")),
        (("--binary",), dict(action="store_true"))]),
)


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="blockinv", description="Blockwise dense-matrix inversion toolkit (B200)")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, help_text, handler, options in _COMMANDS:
        p = sub.add_parser(name, help=help_text)
        for flags, kwargs in options:
            p.add_argument(*flags, **kwargs)
        p.set_defaults(fn=handler)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (BlockInvError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return next(c for kinds, c in _EXIT_MAP if isinstance(exc, kinds))


if __name__ == "__main__":
    sys.exit(main())
