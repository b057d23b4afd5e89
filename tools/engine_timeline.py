"""Per-lane step timeline of the engine on the bench workload (cfg2, batch 4),
from timing events the engine records after every step inside its CUDA graph
(BI_ENGINE_TIMELINE=1).  Prints, per lane, the end time of every step and its
duration (end minus the previous step's end on that lane).

  python tools/engine_timeline.py [--schedule eq7|pivot_a] [--reps 3]
"""
import argparse
import os
import sys
from pathlib import Path

os.environ["BI_ENGINE_TIMELINE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200 import _lib  # noqa: E402
from paper_2305_11103_b200.engine import decode_step, loopid_for_step  # noqa: E402
from paper_2305_11103_b200.workloads import cfg2, cfg4  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--schedule", default="eq7")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--host", action="store_true", help="time the host-buffer path (run_host, pinned)")
    ap.add_argument("--cfg", type=int, default=2, choices=(2, 4), help="2: batch of 4 x 4096; 4: one 16384")
    ap.add_argument("--summary", action="store_true", help="per step kind totals instead of every step")
    args = ap.parse_args()
    if args.cfg == 2:
        ms, sizes = cfg2(4)
    else:
        m, sizes = cfg4()
        ms = m[None]
    eng = bi.DeviceEngine(sizes, batch=ms.shape[0], schedule=args.schedule)
    eng.load(ms)
    if args.host:
        pin_in = torch.from_numpy(ms).pin_memory()
        pin_out = torch.empty_like(pin_in).pin_memory()
        run = lambda: eng.run_host(pin_in.numpy(), pin_out.numpy())  # noqa: E731
    else:
        run = eng.run
    for _ in range(args.reps):
        run()
    eng.check()
    nl = min(int(os.environ.get("BI_ENGINE_LANES", "8")), ms.shape[0])
    ns = eng.n_steps
    buf = (_lib.ctypes.c_float * (nl * (ns + 1)))()
    _lib.check(_lib.lib().bi_engine_timeline(eng._h, buf), "bi_engine_timeline")
    t = np.array(buf[:], dtype=np.float64).reshape(nl, ns + 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    print(f"schedule {args.schedule}: run {e0.elapsed_time(e1):.2f} ms; per-lane step end (duration) in ms")
    kinds = []
    for st in range(1, ns + 1):
        if args.schedule != "eq7":
            kinds.append("all")
            continue
        a = decode_step(loopid_for_step(st, len(sizes)))
        if a.kind == "diag":
            kinds.append("D")
        elif a.kind == "arrows_and_schur" or a.sid is not None:
            kinds.append(f"A{a.sid}")
        else:
            kinds.append(f"D+U{a.depth}")
    if args.summary:
        for l in range(nl):
            tot = {}
            prev = 0.0
            for st in range(1, ns + 1):
                k = kinds[st - 1]
                c = tot.setdefault(k, [0, 0.0])
                c[0] += 1
                c[1] += t[l, st] - prev
                prev = t[l, st]
            print(f"L{l}: " + "; ".join(f"{k} x{c[0]} {c[1]:.2f} ms ({c[1] / c[0]:.3f})" for k, c in sorted(tot.items())))
        for mask, name in ((1, "GEMM ops only"), (2, "leaf inversions only")):
            for _ in range(2):
                eng.run_phase(mask)
            e0.record()
            eng.run_phase(mask)
            e1.record()
            torch.cuda.synchronize()
            print(f"{name}: {e0.elapsed_time(e1):.2f} ms")
        return
    print("step " + " ".join(f"{k:>13s}" for k in kinds))
    for l in range(nl):
        row = []
        prev = None
        for st in range(1, ns + 1):
            end = t[l, st]
            dur = end - prev if prev is not None else end
            row.append(f"{end:6.2f}({dur:5.2f})")
            prev = end
        print(f"L{l}   " + " ".join(row))


if __name__ == "__main__":
    main()
