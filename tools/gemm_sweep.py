"""K1 (bi_gemm) vs cuBLAS DGEMM (torch float64, measurement only) on the
engine's shapes.  Usage: python tools/gemm_sweep.py [--profile SHAPE]"""

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_11103_b200 import _lib  # noqa: E402

SHAPES = [  # (m, n, k, batch, accumulate)
    (512, 512, 512, 32, False),
    (1024, 1024, 1024, 16, False),
    (2048, 2048, 2048, 8, False),
    (2048, 2048, 2048, 8, True),
    (4096, 4096, 4096, 1, False),
    (8192, 8192, 8192, 1, False),
    (512, 480, 32, 32, True),  # old K3 trailing update
    (512, 96, 32, 32, True),   # K3 inner update
    (512, 384, 128, 32, True),  # K3 outer update
    (256, 256, 256, 64, False),
    (512, 96, 32, 8, True),    # K3 inner update, 8 leaves
    (512, 384, 128, 8, True),  # K3 outer update, 8 leaves
    (128, 128, 16, 1, False),  # one tile, one k-tile: launch + pipeline latency
]


def run_k1(a, b, c, d, batch, neg=False):
    L = _lib.lib()
    m, k = a.shape[-2:]
    n = b.shape[-1]
    rc = L.bi_gemm(m, n, k, -1 if neg else 1, a.data_ptr(), a.stride(-2), a.stride(0) if a.dim() == 3 else 0,
                   b.data_ptr(), b.stride(-2), b.stride(0) if b.dim() == 3 else 0,
                   c.data_ptr() if c is not None else None, c.stride(-2) if c is not None else 0,
                   (c.stride(0) if c is not None and c.dim() == 3 else 0),
                   d.data_ptr(), d.stride(-2), d.stride(0) if d.dim() == 3 else 0, batch, _lib.stream_ptr())
    assert rc == 0, L.bi_last_error()


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", type=int, default=-1, help="run only shape index once (for ncu)")
    args = ap.parse_args()
    _lib.load_library()
    shapes = SHAPES if args.profile < 0 else [SHAPES[args.profile]]
    for (m, n, k, batch, accum) in shapes:
        a = torch.randn(batch, m, k, dtype=torch.float64, device="cuda")
        b = torch.randn(batch, k, n, dtype=torch.float64, device="cuda")
        c = torch.randn(batch, m, n, dtype=torch.float64, device="cuda") if accum else None
        d = torch.empty(batch, m, n, dtype=torch.float64, device="cuda")
        flops = 2.0 * m * n * k * batch
        if args.profile >= 0:
            run_k1(a, b, c, d, batch)
            torch.cuda.synchronize()
            continue
        t1 = timeit(lambda: run_k1(a, b, c, d, batch))
        ref = (c if accum else 0) + torch.bmm(a, b)
        err = (d - ref).norm() / ref.norm()
        t2 = timeit(lambda: torch.baddbmm(c, a, b) if accum else torch.bmm(a, b))
        print(f"{m}x{n}x{k} b{batch} acc={accum}: K1 {flops / t1 / 1e9:6.2f} TF/s ({t1 * 1e3:8.1f} us)  "
              f"cuBLAS {flops / t2 / 1e9:6.2f} TF/s ({t2 * 1e3:8.1f} us)  relerr {err:.1e}", flush=True)


if __name__ == "__main__":
    main()
