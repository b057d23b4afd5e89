"""Native column-sharded scheduler on ONE B200: cfg4 (n=16384,
64 x 256) through bi_shard_group_run with P ranks mapped to the same GPU,
against the single-device engine.  P = 1 measures the segment driver's
overhead (graph per segment, no exchanges); P > 1 adds the exchanges (device
-local copies here) and runs the ranks' segments concurrently on one GPU --
a schedule check, not a scaling number (one GPU).

    python tools/shard_bench.py [--reps 5] [--ps 1,2,4,8]
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200 import shard  # noqa: E402
from paper_2305_11103_b200.workloads import cfg4  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ps", default="1,2,4,8")
    args = ap.parse_args()
    m, sizes = cfg4()
    eng = bi.DeviceEngine(sizes)
    eng.load(m)
    t_single = timed(eng.run, args.reps)
    eng.check()
    ref = eng.Minv[0, :, :m.shape[0]].cpu().numpy()
    del eng
    bi.release_engines()
    out = {"single_engine_ms": t_single}
    for P in [int(x) for x in args.ps.split(",")]:
        shards = []
        for r in range(P):
            sh = shard.NativeShard(sizes, P, r)
            sh.load(m)
            shards.append(sh)
        torch.cuda.synchronize()
        t = timed(lambda: shard.run_group(shards), args.reps)
        fail = shard.first_singular([sh.check() for sh in shards])
        res = np.empty_like(m)
        for sh in shards:
            sh.write_slab(res)
        out[f"P{P}"] = {"ms": t, "vs_single": t / t_single, "bitwise_equal": bool(np.array_equal(res, ref)),
                        "singular": fail, "segments": len(shards[0].segments()),
                        "exchanges": shards[0].n_xchg, "launches_per_rank": shards[0].launches()}
        del shards
        torch.cuda.empty_cache()
        print(json.dumps({f"P{P}": out[f"P{P}"]}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
