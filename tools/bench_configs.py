"""Time the other BASELINE.json configs on one B200 (not the driver's bench
line; recorded under profiles/).  Each run is verified by the on-device
residual ||A X - I||_F (K1 + K4).

  cfg1  n=512, (256, 256): invertor_inplace_by_a and run_inversion
  cfg3  n=6000, split 1000, singular A11: invert_with_fallback -> via_d
  cfg4  n=16384, 64 x 256 blocks: run_inversion step engine (127 steps)
  cfg5  n=65536, 256 x 256 blocks (--cfg5): run_inversion on ONE GPU
        (~138 GB of device state); the config's own seed-5 NumPy stream
        (workloads.cfg5), plus one end-to-end run_inversion on the NumPy array
  cfg4 and cfg5 also run the opt-in schedule="pivot_a" (2n^3 block-level
  invertor_by_a recursion).
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200 import workloads  # noqa: E402
from paper_2305_11103_b200.core import _residual_device  # noqa: E402


def events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def time_engine(eng, reps):
    eng.run()
    eng.check()
    torch.cuda.synchronize()
    a, b = events()
    a.record()
    for _ in range(reps):
        eng.run()
    b.record()
    torch.cuda.synchronize()
    eng.check()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg5", action="store_true")
    ap.add_argument("--skip", default="")
    args = ap.parse_args()
    out = {}
    skip = set(args.skip.split(","))

    if "cfg1" not in skip:
        m, sizes = workloads.cfg1()
        x = m.copy()
        bi.invertor_inplace_by_a(x)
        t0 = time.perf_counter()
        for _ in range(5):
            x = m.copy()
            bi.invertor_inplace_by_a(x)
        t_inplace = (time.perf_counter() - t0) / 5
        eng = bi.DeviceEngine(sizes, 1)
        eng.load(m)
        ms = time_engine(eng, 20)
        fro, _ = _residual_device(eng.M, eng.Minv, batch=True)
        out["cfg1"] = {"inplace_by_a_s_e2e": t_inplace, "run_inversion_device_ms": ms,
                       "tflops_nominal_device": 2 * 512**3 / (ms * 1e-3) / 1e12,
                       "residual_fro": float(fro[0]), "residual_fro_inplace": bi.residual_frobenius(m, x)}
        print("cfg1", out["cfg1"], flush=True)

    if "cfg3" not in skip:
        m, split = workloads.cfg3()
        res = np.empty_like(m)
        bi.invert_with_fallback(m, split, res)
        from paper_2305_11103_b200 import _lib
        from paper_2305_11103_b200.schur import schur2x2_device

        md = _lib.to_device(m)
        od = _lib.empty_matrix(6000, 6000)
        schur2x2_device("D", md, split, od)
        torch.cuda.synchronize()
        a, b = events()
        a.record()
        for _ in range(3):
            schur2x2_device("D", md, split, od)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        out["cfg3"] = {"via": bi.invert_with_fallback(m, split, res), "via_d_device_ms": ms,
                       "tflops_nominal": 2 * 6000**3 / (ms * 1e-3) / 1e12,
                       "residual_fro": bi.residual_frobenius(m, res)}
        print("cfg3", out["cfg3"], flush=True)

    if "cfg4" not in skip:
        m, sizes = workloads.cfg4()
        for sched in ("eq7", "pivot_a"):
            eng = bi.DeviceEngine(sizes, 1, schedule=sched)
            eng.load(m)
            ms = time_engine(eng, 2)
            fro, _ = _residual_device(eng.M, eng.Minv, batch=True)
            c = eng.counters()
            key = "cfg4" if sched == "eq7" else "cfg4_pivot_a"
            out[key] = {"run_inversion_device_ms": ms, "tflops_nominal": 2 * 16384**3 / (ms * 1e-3) / 1e12,
                        "tflops_algorithmic": (c["gemm_flops"] + c["leaf_flops"]) / (ms * 1e-3) / 1e12,
                        "residual_fro": float(fro[0]), "schedule": sched}
            print(key, out[key], flush=True)
            del eng
            torch.cuda.empty_cache()
        del m

    if args.cfg5:
        n = 65536
        m5, sizes = workloads.cfg5()  # the config's own seed-5 NumPy stream, 34 GB
        for sched in ("eq7", "pivot_a"):
            torch.cuda.reset_peak_memory_stats()
            eng = bi.DeviceEngine(sizes, 1, schedule=sched)
            eng.load(m5)
            torch.cuda.synchronize()
            ms = time_engine(eng, 1)
            fro, mx = _residual_device(eng.M, eng.Minv, batch=True)
            key = "cfg5" if sched == "eq7" else "cfg5_pivot_a"
            out[key] = {"run_inversion_device_s": ms / 1e3, "tflops_nominal": 2 * n**3 / (ms * 1e-3) / 1e12,
                        "residual_fro": float(fro[0]), "residual_max": float(mx[0]),
                        "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9, "schedule": sched,
                        "input": "workloads.cfg5(): N(0,1)/256 + 4I from numpy default_rng(5)"}
            print(key, out[key], flush=True)
            del eng
            bi.release_engines()
        t0 = time.perf_counter()
        x = bi.run_inversion(m5, sizes=sizes).store.data  # end to end, NumPy in / NumPy out
        out["cfg5_e2e_s"] = time.perf_counter() - t0
        print("cfg5 e2e run_inversion", out["cfg5_e2e_s"], "s", flush=True)
        del x
        bi.release_engines()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
