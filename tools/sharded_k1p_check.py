"""The thread-per-GPU sharded schedule at a larger size, with gathered copies
(BI_FUSED_GATHER=0) and with K1P (1, cluster sizes 1 and 4), on ranks that
share one B200: bitwise equal to the single-device engine, plus host wall
times (not a scaling number: every "GPU" here is the same device).

    python tools/sharded_k1p_check.py [n] [block]
"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200.distributed import run_inversion_local  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    sizes = [b] * (n // b)
    g = np.random.default_rng(4)
    m = g.standard_normal((n, n)) / np.sqrt(n)
    m[np.diag_indices(n)] += 4.0
    t0 = time.perf_counter()
    single = bi.run_inversion(m, sizes=sizes).to_dense()
    print(f"n={n} blocks={len(sizes)}x{b}: single device {time.perf_counter() - t0:.2f} s "
          f"residual {bi.residual_norm(m, single):.2e}", flush=True)
    for gpus in (2, 4):
        for fused in ("0", "1"):
            os.environ["BI_FUSED_GATHER"] = fused
            t0 = time.perf_counter()
            out = run_inversion_local(m, sizes, gpus, devices=[0] * gpus)
            dt = time.perf_counter() - t0
            print(f"  {gpus} ranks on one B200, fused={fused}: {dt:.2f} s, bitwise equal: "
                  f"{np.array_equal(out, single)}", flush=True)


if __name__ == "__main__":
    main()
