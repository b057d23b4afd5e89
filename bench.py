"""Benchmark: FP64 blockwise inversion on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): a batch of 4 independent
n=4096 float64 matrices, each N(0,1)/sqrt(n) + 2I (seeds [2, b]), partitioned
into 8 diagonal blocks of order 512, inverted by the reference's step engine
(run_inversion, 15 steps: recursive halving 8 -> 4 -> 2).  One bench "step"
= one inversion of the whole batch.

  value  : whole-job FP64 TFLOP/s at 2n^3 nominal per inverse, inputs already
           resident in HBM, device-timed with CUDA events (max over ranks).
  e2e    : the same metric through the public API run_inversion_batch() with
           page-locked host buffers: H2D of the 4 inputs, the inversion, D2H of
           the 4 inverses inside the timed region.
  roofline: the dominant kernel K1 (gemm_tma_refill_kernel<4, 64>, FP64 tensor pipe): its
           algorithmic flops over its own device time (engine GEMM ops run
           alone), against the measured DMMA peak (MEASURED_PEAKS.json has no
           FP64 entry; profiles/r01_fp64_dmma_dfma_microbench.txt).
  cpu_baseline: the reference CPU algorithm (oracle/ port, op-for-op the
           reference) on a bounded sample (rank 0, N=1).

Multi-GPU: one process per GPU (torchrun); the batch is replicated per rank
(independent matrices, no data-path collective) -> "scaling": "weak".

--impl reference: times the reference CPU implementation (the oracle port --
the Python reference cannot travel to the GPU box) on the host cores, same
metric/config, each step a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N = 4096
NBLOCKS = 8
BATCH = 4
METRIC = "FP64 inversion TFLOP/s (2n^3 nominal) and s/inverse, 1/2/4/8 B200 vs CPU ref"
UNIT = "TFLOP/s"
WORKLOAD = "cfg2: batch of 4 x n=4096 float64, 8 diagonal blocks of 512, run_inversion step engine"
# measured DMMA.8x8x4 chip peak on this pool's B200 (profiles/r01_fp64_dmma_dfma_microbench.txt)
FP64_PEAK_TFLOPS = 36.98
FP64_PEAK_SOURCE = "measured: DMMA.8x8x4 microbench 36.98 TF/s (profiles/r01_fp64_dmma_dfma_microbench.txt); " \
                   "MEASURED_PEAKS.json has no FP64 entry; cuBLAS DGEMM 8192^3 = 35.47 TF/s"
# CPU sample for the reference arm / cpu_baseline: same 8-block structure, scaled down
SAMPLE_N = 1024
SAMPLE_SIZES = [128] * 8


def nominal_flops(n: int) -> float:
    return 2.0 * float(n) ** 3


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference (oracle port of the reference algorithm)
# ---------------------------------------------------------------------------


def _ref_sample_worker(seed: int) -> float:
    import oracle

    g = np.random.default_rng([2, 1000 + seed])
    m = g.standard_normal((SAMPLE_N, SAMPLE_N)) / np.sqrt(SAMPLE_N)
    m[np.diag_indices(SAMPLE_N)] += 2.0
    t0 = time.perf_counter()
    oracle.run_inversion(m, sizes=SAMPLE_SIZES)
    return time.perf_counter() - t0


def _ref_warm(_: int) -> None:
    import oracle

    g = np.random.default_rng(0)
    oracle.run_inversion(g.standard_normal((64, 64)) + 64 * np.eye(64), sizes=[8] * 8)


def host_threads() -> int:
    """Host threads this process may run on (affinity-aware)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def sample_count(procs: int) -> int:
    """Sample matrices per step: the batch, widened to keep every process busy."""
    return max(BATCH, procs)


def reference_pool(procs: int):
    """Worker processes for the reference arm, started outside the timed
    region (None for a single process)."""
    import multiprocessing as mp

    return mp.get_context("fork").Pool(procs) if procs > 1 else None


def reference_sample_step(procs: int, pool=None) -> tuple[float, float]:
    """Invert sample_count(procs) sample matrices with the reference
    algorithm, `procs` processes in parallel, one matrix per process at a
    time (the reference engine itself is single-threaded: its per-k ufunc
    loop is GIL-bound), so the arm uses every host thread.
    Returns (wall seconds, nominal flops)."""
    count = sample_count(procs)
    own = pool is None and procs > 1
    if own:
        pool = reference_pool(procs)
    try:
        t0 = time.perf_counter()
        if pool is None:
            for b in range(count):
                _ref_sample_worker(b)
        else:
            pool.map(_ref_sample_worker, range(count), chunksize=1)
        return time.perf_counter() - t0, count * nominal_flops(SAMPLE_N)
    finally:
        if own:
            pool.close()


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    procs = host_threads()
    for _ in range(args.warmup):  # untimed warm-up: tiny problem (imports, page-in)
        import oracle

        g = np.random.default_rng(0)
        m = g.standard_normal((64, 64)) + 64 * np.eye(64)
        oracle.run_inversion(m, sizes=[8] * 8)
    times = []
    flops = 0.0
    pool = reference_pool(procs)
    try:
        if pool is not None:
            pool.map(_ref_warm, range(procs), chunksize=1)  # workers forked and numpy paged in
        for _ in range(args.steps):
            dt, flops = reference_sample_step(procs, pool)
            times.append(dt)
    finally:
        if pool is not None:
            pool.close()
    total = sum(times)
    value = flops * args.steps / total / 1e12
    sample = (f"{sample_count(procs)} matrices of n={SAMPLE_N} (8 blocks of {SAMPLE_SIZES[0]}, same generator family) per step, "
              f"reference run_inversion algorithm (oracle/ port, op-for-op), {procs} processes")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample_n": SAMPLE_N, "batch": BATCH},
        "s_per_inverse": total / (args.steps * sample_count(procs)),
        "s_per_inverse_n4096_extrapolated_n3": total / (args.steps * sample_count(procs)) * (N / SAMPLE_N) ** 3,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def _load_traffic() -> float | None:
    p = ROOT / "profiles" / "r01_ncu_gemm_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def run_gpu_arm(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2305_11103_b200 import build_native

    if build_native.needs_build():
        build_native.build()
    import paper_2305_11103_b200 as bi
    from paper_2305_11103_b200.workloads import cfg2

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    ms, sizes = cfg2(BATCH, N, NBLOCKS)
    eng = bi.DeviceEngine(sizes, batch=BATCH)
    eng.load(ms)
    stream = torch.cuda.current_stream()

    # correctness gate (untimed): residual of every inverse on the device
    eng.run()
    eng.check()
    from paper_2305_11103_b200.core import _residual_device

    fro, mx = _residual_device(eng.M, eng.Minv, batch=True)
    assert np.all(fro <= 1e-9 * N), fro

    for _ in range(args.warmup):
        eng.run()
    torch.cuda.synchronize()

    # ---- timed region: K steps, inputs resident in HBM (> L2: 4 x 128 MiB in + out)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            eng.run()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    eng.check()
    minv_ref = eng.Minv.cpu().numpy()  # phase timing below overwrites M_inv
    ms_total = ev0.elapsed_time(ev1)
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = world * BATCH * nominal_flops(N) / (ms_step * 1e-3) / 1e12
    counters = eng.counters()
    alg_flops = counters["gemm_flops"] + counters["leaf_flops"]
    launches = eng.launches()

    # ---- per-kernel: engine K1 GEMM ops alone and leaf inversions alone
    def time_phase(mask: int, reps: int) -> float:
        for _ in range(2):
            eng.run_phase(mask)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            eng.run_phase(mask)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    reps = max(3, min(args.steps, 10))
    gemm_ms = time_phase(1, reps)
    leaf_ms = time_phase(2, reps)
    k1_tflops = counters["gemm_flops"] / (gemm_ms * 1e-3) / 1e12

    # ---- the opt-in 2n^3 pivot-A schedule on the same inputs:
    # reported beside the headline, which stays on the reference's Eq. 7 engine
    pa = bi.DeviceEngine(sizes, batch=BATCH, schedule="pivot_a")
    pa.load(ms)
    pa.run()
    pa.check()
    pa_fro, _ = _residual_device(pa.M, pa.Minv, batch=True)
    assert np.all(pa_fro <= 1e-9 * N), pa_fro
    for _ in range(args.warmup):
        pa.run()
    torch.cuda.synchronize()
    barrier()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        pa.run()
    p1.record(stream)
    torch.cuda.synchronize()
    pa.check()
    tp = torch.tensor([p0.elapsed_time(p1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tp, op=dist.ReduceOp.MAX)
    pa_ms_step = float(tp.item()) / args.steps
    pa_c = pa.counters()
    pivot_a = {"value": world * BATCH * nominal_flops(N) / (pa_ms_step * 1e-3) / 1e12, "unit": UNIT,
               "ms_per_step": pa_ms_step,
               "algorithmic_tflops": world * (pa_c["gemm_flops"] + pa_c["leaf_flops"]) / (pa_ms_step * 1e-3) / 1e12,
               "residual_fro_max": float(np.max(pa_fro)),
               "note": "opt-in schedule='pivot_a' (block-level invertor_by_a recursion, 2n^3 flops); "
                       "not the reference's run_inversion step schedule"}
    del pa

    # ---- e2e through the public API with page-locked host buffers
    pin_in = torch.from_numpy(ms).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    in_np, out_np = pin_in.numpy(), pin_out.numpy()
    for _ in range(max(1, min(args.warmup, 3))):
        bi.run_inversion_batch(in_np, sizes, out=out_np)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        bi.run_inversion_batch(in_np, sizes, out=out_np)
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms_step = float(te.item()) / args.steps
    e2e_value = world * BATCH * nominal_flops(N) / (e2e_ms_step * 1e-3) / 1e12
    assert np.array_equal(out_np, minv_ref)  # the API path computes the same inverses

    # ---- CPU baseline (rank 0, N=1): reference algorithm on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        procs = host_threads()
        # bounded sample, repeated to >= 10 s of CPU work (at most 8 rounds)
        dt, fl, rounds = 0.0, 0.0, 0
        pool = reference_pool(procs)
        try:
            if pool is not None:
                pool.map(_ref_warm, range(procs), chunksize=1)
            while rounds < 8 and (rounds == 0 or dt < 10.0):
                d1, f1 = reference_sample_step(procs, pool)
                dt, fl, rounds = dt + d1, fl + f1, rounds + 1
        finally:
            if pool is not None:
                pool.close()
        cpu = {"value": fl / dt / 1e12, "unit": UNIT, "cores": procs, "kind": "port",
               "sample": f"{rounds} x {sample_count(procs)} matrices n={SAMPLE_N} (8 blocks of {SAMPLE_SIZES[0]}) through the "
                         f"reference run_inversion algorithm (oracle/ port, op-for-op), {procs} processes, "
                         f"{dt:.1f} s"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": N, "blocks": sizes, "batch_per_gpu": BATCH,
                       "parallelism": f"replicas x{world}", "l2": "inputs larger than L2 (1 GiB in+out per step)"},
            "s_per_inverse": ms_step * 1e-3 / BATCH,
            "algorithmic_tflops": world * alg_flops / (ms_step * 1e-3) / 1e12,
            "frac_of_fp64_peak_nominal": value / world / FP64_PEAK_TFLOPS,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(ms.nbytes),
                    "d2h_bytes_per_step": int(ms.nbytes), "ms_per_step": e2e_ms_step,
                    "api": "paper_2305_11103_b200.run_inversion_batch (pinned host buffers)"},
            "roofline": {"bound": "tensor", "achieved": k1_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": k1_tflops / FP64_PEAK_TFLOPS, "traffic": _load_traffic(),
                         "kernel": "gemm_tma_refill_kernel<4, 64> (K1 TMA feeder, engine GEMM ops)", "peak_source": FP64_PEAK_SOURCE,
                         "kernel_ms_per_step": gemm_ms, "kernel_flops_per_step": counters["gemm_flops"],
                         "share_of_step": gemm_ms / ms_step,
                         "leaf_inversion_ms_per_step": leaf_ms,
                         "leaf_inversion_tflops": counters["leaf_flops"] / (leaf_ms * 1e-3) / 1e12},
            "gpu_launches": launches["total"] * args.steps,
            "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
            "residual_fro_max": float(np.max(fro)),
        }
        line["pivot_a_schedule"] = pivot_a
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
