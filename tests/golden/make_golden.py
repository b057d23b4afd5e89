"""Generate tests/golden/golden.npz by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

The fixtures pin the CPU oracle (oracle/) to the reference's actual outputs
and pin the product's host logic (partition, step schedule, counters).  Every
input is regenerated from its seed by the tests; only reference OUTPUTS are
stored.  Nothing here is read at run time on the GPU box except the .npz.
"""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden.npz"


def well_conditioned(order, seed):
    g = np.random.default_rng(seed)
    m = g.uniform(-1.0, 1.0, (order, order))
    m[np.diag_indices(order)] += 2.0 * order
    return m


def cfg3_small(n=120, split=20, rank=10):
    rng = np.random.default_rng(3)
    m = rng.standard_normal((n, n))
    u = rng.standard_normal((split, rank))
    v = rng.standard_normal((split, rank))
    m[:split, :split] = u @ v.T
    m[split:, split:] += float(n) * np.eye(n - split)
    return m


# (name, sizes or None for the default partition, order, seed)
ENGINE_CASES = [
    ("def2", None, 2, 602), ("def3", None, 3, 603), ("def5", None, 5, 605), ("def9", None, 9, 609),
    ("def12", None, 12, 612), ("def21", None, 21, 621), ("def33", None, 33, 633), ("def64", None, 64, 664),
    ("s5_7", [5, 7], 12, 43), ("s3_9_5_11", [3, 9, 5, 11], 28, 44), ("s8x8", [8] * 8, 64, 45),
    ("s16x4", [16] * 4, 64, 46), ("s6x16", [6] * 16, 96, 47),
]


def main():
    sys.path.insert(0, str(REF_SRC))
    import blockinv as R
    from blockinv.core import release_mode
    from blockinv.engine import decode_step, loopid_for_step, step_plan, total_steps, updown_iteration_map
    from blockinv.partition import make_partition
    from blockinv.storage import load_minv_store, load_tsets

    g = {}
    # --- schedule tables (engine.py:73-170) for blocksizes 1..64
    for bs in (1, 2, 4, 8, 16, 32, 64):
        rows = []
        for s in range(1, total_steps(bs) + 1):
            p = step_plan(s, bs)
            a = p.action
            kind = {"invert_diagonals": 0, "arrows_and_schur": 1, "schur_diag_and_assemble": 2}[a.kind]
            rows.append(list(p.loopid) + [kind, 1 if a.source == "tset" else 0,
                                          -1 if a.cid is None else a.cid, -1 if a.sid is None else a.sid,
                                          a.depth])
        g[f"plan_{bs}"] = np.array(rows, dtype=np.int64)
    g["updown_16"] = np.array([[updown_iteration_map(r, c) for c in range(1, 17)] for r in range(1, 17)])
    # --- default partitions (partition.py:63-84)
    orders = list(range(2, 200)) + [333, 1024, 2047, 4096, 10000]
    g["partition_orders"] = np.array(orders)
    g["partition_sizes"] = np.concatenate([np.array(make_partition(o).sizes) for o in orders])
    with release_mode():
        # --- engine outputs + counters
        for name, sizes, order, seed in ENGINE_CASES:
            m = well_conditioned(order, seed)
            c = R.OpCounters()
            g[f"engine_{name}"] = R.run_inversion(m, sizes=sizes, counters=c).to_dense()
            g[f"engine_{name}_counters"] = np.array([c.multiplies, c.inversions, c.reductions])
        # --- per-step state for [8]*8 (checkpoint hook, engine.py:536-539)
        sizes = [8] * 8
        m = well_conditioned(64, 45)
        scheme = R.partition_from_sizes(sizes)
        for step in range(1, total_steps(8) + 1):
            with tempfile.TemporaryDirectory() as d:
                R.run_inversion(m, sizes=sizes, checkpoint_dir=d, stop_after_step=step)
                g[f"step8x8_minv_{step}"] = load_minv_store(d, scheme, False).to_dense()
                if step == total_steps(8):
                    ts = load_tsets(d, scheme, False)
                    for lv, t in ts.items():
                        for nm, arr in t.entries():
                            g[f"step8x8_tset_{lv}_{nm}"] = arr
        # --- a checkpoint directory written by the reference (format parity,
        #     SURVEY 8f #3): [8]*4, stopped after step 4 of 7; every file's bytes
        for stop in (4,):
            with tempfile.TemporaryDirectory() as d:
                mc = well_conditioned(32, 61)
                R.run_inversion(mc, sizes=[8] * 4, checkpoint_dir=d, stop_after_step=stop)
                for path in sorted(Path(d).rglob("*")):
                    if path.is_file():
                        key = "ckpt4_file__" + str(path.relative_to(d)).replace("/", "__")
                        g[key] = np.frombuffer(path.read_bytes(), dtype=np.uint8).copy()
            g["ckpt4_final"] = R.run_inversion(mc, sizes=[8] * 4).to_dense()
        # --- recursive procedures and the GJ oracle
        for order in (8, 17, 64):
            m = well_conditioned(order, 30 + order)
            g[f"by_a_{order}"], _ = R.invertor_by_a(m)
            x = m.copy()
            R.invertor_inplace_by_a(x)
            g[f"inplace_{order}"] = x
            g[f"gj_{order}"] = R.gauss_jordan_oracle(m)
        # --- formulas
        m = well_conditioned(60, 3)

        def gj_sub(b, o):
            o[...] = R.gauss_jordan_oracle(b)

        for nm, f in (("a", R.invert_via_a), ("d", R.invert_via_d), ("ad", R.invert_via_ad)):
            o = np.empty((60, 60))
            f(R.diagonal_quad(m, 25), gj_sub, o)
            g[f"via_{nm}_60_25"] = o
        for order, split in ((8, 4), (7, 3)):
            m = well_conditioned(order, 10)
            for nm, f in (("b", R.invert_via_b), ("c", R.invert_via_c), ("bc", R.invert_via_bc)):
                o = np.empty((order, order))
                f(R.counterdiagonal_quad(m, split), R.invert_small, o)
                g[f"via_{nm}_{order}_{split}"] = o
        perm2 = np.array([[0.0, 1.0], [1.0, 0.0]])
        o = np.empty((2, 2))
        g["fallback_perm2_name"] = np.array([R.invert_with_fallback(perm2, 1, o)])
        g["fallback_perm2_out"] = o
        m = well_conditioned(4, 20)
        m[0, 0] = 0.0
        o = np.empty((4, 4))
        g["fallback_kat_name"] = np.array([R.invert_with_fallback(m, 1, o)])
        g["fallback_kat_out"] = o
        # --- cfg3 construction, scaled: singular A11 -> via_d with the pivoted sub
        m3 = cfg3_small()
        o = np.empty_like(m3)
        R.invert_via_d(R.diagonal_quad(m3, 20), gj_sub, o)
        g["cfg3s_via_d_gj"] = o
        try:
            R.gauss_jordan_oracle(m3[:20, :20])
            g["cfg3s_a11_singular"] = np.array([0])
        except R.core.SingularMatrix if hasattr(R.core, "SingularMatrix") else Exception:
            g["cfg3s_a11_singular"] = np.array([1])
        # --- invertor_by_ad / invertor_with_fallback (recursive.py:366-496)
        for order in (8, 17, 64):
            m = well_conditioned(order, 30 + order)
            c = R.OpCounters()
            g[f"by_ad_{order}"], _ = R.invertor_by_ad(m, c)
        for order in (6, 16):
            c = R.OpCounters()
            g[f"fallback_rec_perm{order}"], _ = R.invertor_with_fallback(np.eye(order)[::-1].copy(), c)
        # --- bench harness (bench.py): generators, CSV text, slope fit; text matrix file bytes
        import importlib

        RB = importlib.import_module("blockinv.bench")
        from blockinv.core import save_text

        for kind in RB.KINDS:
            for order in (1, 5, 12):
                g[f"gen_{kind}_{order}"] = RB.generate(order, seed=7, kind=kind)
        recs = [RB.TimingRecord("a", o, 1, 1e-3 * (o / 8.0) ** 2.9 * (1.0 + 0.03 * ((o * 7) % 5)), 1e-13 * o)
                for o in (8, 16, 32, 64, 128)]
        fit = RB.fit_slope(recs, 8, 128)
        g["bench_fit"] = np.array([fit.exponent, fit.stderr, fit.n_points])
        g["bench_csv"] = np.frombuffer(RB.records_to_csv(recs).encode(), dtype=np.uint8).copy()
        with tempfile.TemporaryDirectory() as d:
            save_text(well_conditioned(3, 5), Path(d) / "m.txt")
            g["text_file_3"] = np.frombuffer((Path(d) / "m.txt").read_bytes(), dtype=np.uint8).copy()
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
