"""K1P (bi_gemm_kseg) vs K1 (bi_gemm on the gathered operand) on one B200.

The segments are local here (one GPU is reachable); on an 8-GPU box they are
the peers' slabs read over NVLink.  Prints, per shape, the kernel rate of
K1P, of K1 on the pre-gathered operand, and of gather (device copies) + K1 --
the sequence the fused path replaces.  CUDA events on the launching stream.
"""

import sys

import torch

sys.path.insert(0, ".")
from paper_2305_11103_b200 import _lib  # noqa: E402
from paper_2305_11103_b200.core import device_gemm, device_gemm_kseg  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    _lib.require_device()
    g = torch.Generator(device="cuda").manual_seed(0)
    for m, n, nseg, w in [(4096, 2048, 4, 1024), (8192, 4096, 8, 1024), (16384, 2048, 8, 2048), (2048, 1024, 2, 1024)]:
        k = nseg * w
        segs = [torch.randn((m, w), dtype=torch.float64, device="cuda", generator=g) for _ in range(nseg)]
        b = torch.randn((k, n), dtype=torch.float64, device="cuda", generator=g)
        d = torch.empty((m, n), dtype=torch.float64, device="cuda")
        gathered = torch.empty((m, k), dtype=torch.float64, device="cuda")
        flops = 2.0 * m * n * k

        def gather():
            for i, s in enumerate(segs):
                gathered[:, i * w:(i + 1) * w].copy_(s)

        t_p = timed(lambda: device_gemm_kseg(segs, b, d))
        gather()
        t_1 = timed(lambda: device_gemm(gathered, b, d))
        t_g = timed(lambda: (gather(), device_gemm(gathered, b, d)))
        print(f"m={m} n={n} k={k} ({nseg} segs): K1P {t_p:.3f} ms {flops / t_p / 1e9:.1f} TF/s | "
              f"K1 gathered {t_1:.3f} ms {flops / t_1 / 1e9:.1f} TF/s | gather+K1 {t_g:.3f} ms "
              f"{flops / t_g / 1e9:.1f} TF/s")


if __name__ == "__main__":
    main()
