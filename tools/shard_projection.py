"""Strong-scaling PROJECTION of the column-sharded level scheduler
from one B200 -- not a multi-GPU measurement.

cfg4 (n = 16384, 64 x 256, Eq. 7) is sharded over P = 1, 2, 4, 8 ranks exactly
as ``bench.py --gpus P`` shards it, and the ranks are run ONE AT A TIME on the
single GPU, segment by segment, with the real exchanges in between (pack ->
the group's send areas copied into each member's receive area -> unpack), so
every rank computes on the real data and the gathered inverse is checked
bitwise against the single engine.  No kernel of one rank ever waits on
another rank's kernel.

Per segment k and rank r the device time t(r, k) of the rank's ops (its
segment graph + pack + unpack) is measured with CUDA events with the GPU to
itself -- what that rank's own GPU would spend.  Ranks run in parallel on a
real box and meet at every exchange, so the projected step is

    T(P) = sum_k max_r t(r, k)  +  sum_exchanges  bytes_received / BW

with BW the assumed all-gather bandwidth per GPU (default 600 GB/s, a
conservative NCCL figure for NVLink 5 / NVSwitch; --bw to change).  The
exchange term is a model; everything else is measured.

    python tools/shard_projection.py [--ps 1,2,4,8] [--reps 3] [--bw 600]
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200 import _lib, shard  # noqa: E402
from paper_2305_11103_b200.workloads import cfg4  # noqa: E402


def run_serial(shards, segs, timed: bool):
    """One full run, the ranks one after the other inside every segment.
    Returns ([k][r] ms of the rank's own work, [k] bytes received per rank)."""
    L = _lib.lib()
    st = _lib.stream_ptr()
    P = len(shards)
    nseg = len(segs[0])
    for sh in shards:
        sh.Minv.zero_()
    times, xbytes = [], []
    for k in range(nseg):
        evs = []
        for r, sh in enumerate(shards):
            b, e, xi = segs[r][k]
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a0.record()
            _lib.check(L.bi_engine_run_ops(sh._h, b, e, 1, st), "bi_engine_run_ops")
            if xi >= 0:
                _lib.check(L.bi_engine_xchg_pack(sh._h, xi, st), "bi_engine_xchg_pack")
            a1.record()
            evs.append([a0, a1])
        recv_bytes = 0
        for r, sh in enumerate(shards):  # the all-gather inside each group, as device copies (not timed)
            xi = segs[r][k][2]
            if xi < 0:
                continue
            x = sh._x[xi]
            chunk = x["rows"] * sh.wmax
            if x["gs"] > 1:
                for m in range(x["g0"], x["g0"] + x["gs"]):
                    src = shards[m]
                    off = sh._recv_off + (m - x["g0"]) * chunk
                    sh._flat[off:off + chunk].copy_(src._flat[src._send_off:src._send_off + chunk])
                recv_bytes = max(recv_bytes, (x["gs"] - 1) * chunk * 8)
        for r, sh in enumerate(shards):
            xi = segs[r][k][2]
            if xi < 0:
                continue
            u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            u0.record()
            _lib.check(L.bi_engine_xchg_unpack(sh._h, xi, st), "bi_engine_xchg_unpack")
            u1.record()
            evs[r] += [u0, u1]
        torch.cuda.synchronize()
        if timed:
            times.append([sum(ev[i].elapsed_time(ev[i + 1]) for i in range(0, len(ev), 2)) for ev in evs])
            xbytes.append(recv_bytes)
    return times, xbytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ps", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--bw", type=float, default=600.0, help="assumed all-gather GB/s received per GPU")
    args = ap.parse_args()
    m, sizes = cfg4()
    n = m.shape[0]
    eng = bi.DeviceEngine(sizes)
    eng.load(m)
    eng.run()
    eng.check()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.reps):
        eng.run()
    b.record()
    torch.cuda.synchronize()
    t1 = a.elapsed_time(b) / args.reps
    ref = eng.Minv[0, :, :n].cpu().numpy()
    del eng
    bi.release_engines()
    print(f"# cfg4 single engine: {t1:.2f} ms")
    print("# P | measured critical path (sum_k max_r) ms | slowest rank's own total ms | exchanges | GB received/rank | "
          f"modelled exchange ms @ {args.bw:.0f} GB/s | projected step ms | projected speed-up | efficiency")
    out = {"single_engine_ms": t1, "bw_gbs": args.bw, "P": {}}
    for P in [int(x) for x in args.ps.split(",")]:
        shards = [shard.NativeShard(sizes, P, r, staging=True) for r in range(P)]
        for sh in shards:
            sh.load(m)
        segs = [sh.segments(1, sh.n_steps) for sh in shards]
        assert len({len(s) for s in segs}) == 1
        run_serial(shards, segs, timed=False)  # graphs captured, caches warm
        res = np.empty_like(m)
        for sh in shards:
            assert sh.check() is None
            sh.write_slab(res)
        assert np.array_equal(res, ref), f"P={P}: serial sharded run differs from the single engine"
        crit, rank_tot, gb = [], [], 0.0
        for _ in range(args.reps):
            times, xbytes = run_serial(shards, segs, timed=True)
            crit.append(sum(max(row) for row in times))
            rank_tot.append(max(sum(row[r] for row in times) for r in range(P)))
            gb = sum(xbytes) / 1e9
        c, rt = min(crit), min(rank_tot)
        nx = sum(1 for s in segs[0] if s[2] >= 0)
        xms = gb / args.bw * 1e3
        proj = c + xms
        print(f"P={P} | {c:8.2f} | {rt:8.2f} | {nx:3d} | {gb:6.2f} | {xms:6.2f} | {proj:8.2f} | {t1 / proj:5.2f}x | "
              f"{t1 / proj / P:5.2f}", flush=True)
        out["P"][P] = {"critical_path_ms": c, "slowest_rank_ms": rt, "exchanges": nx, "gb_received_per_rank": gb,
                       "exchange_ms_model": xms, "projected_ms": proj, "speedup": t1 / proj,
                       "bitwise_equal_to_single_engine": True}
        del shards
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
