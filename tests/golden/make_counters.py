"""Golden OpCounters of the reference's recursive procedures (run HERE, with
the reference importable from /root/reference/pkg/src):
invertor_by_a, invertor_inplace_by_a and invertor_by_ad on seeded
well-conditioned matrices, every OpCounters field.  Writes
tests/golden/counters.json (committed); tests/test_host.py checks the
framework's reported tallies against it.

    python tests/golden/make_counters.py
"""

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

ORDERS = list(range(1, 41)) + [63, 64, 65, 100, 127, 128, 200, 256, 257, 300, 600]


def main() -> None:
    from blockinv.recursive import invertor_by_a, invertor_by_ad, invertor_inplace_by_a

    out = {}
    for n in ORDERS:
        g = np.random.default_rng(5000 + n)
        m = g.uniform(-1.0, 1.0, (n, n))
        m[np.diag_indices(n)] += 2.0 * n
        rec = {}
        _, c = invertor_by_a(m)
        rec["by_a"] = c
        c = invertor_inplace_by_a(m.copy())
        rec["inplace"] = c
        _, c = invertor_by_ad(m)
        rec["by_ad"] = c
        out[str(n)] = {k: {f: getattr(v, f) for f in ("multiplies", "inversions", "reductions", "peak_scratch",
                                                    "schur_scratch", "nodes")} for k, v in rec.items()}
    p = Path(__file__).with_name("counters.json")
    p.write_text(json.dumps(out, indent=0, sort_keys=True))
    print(f"wrote {p} ({len(out)} orders)")


if __name__ == "__main__":
    main()
