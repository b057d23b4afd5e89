"""Benchmark: FP64 blockwise inversion on B200 (BASELINE.json metric).

Headline workload (BASELINE.json configs[3], SURVEY 8d cfg4 -- the config the
metric's 1/2/4/8-GPU figures are quoted on): one n=16384 float64 matrix,
N(0,1)/sqrt(n) + 4I from seed 4, partitioned into 64 diagonal blocks of order
256, inverted by the reference's step engine (run_inversion, Eq. 7 schedule,
127 steps: recursive halving 64 -> 32 -> ... -> 2).  One bench "step" = one
inversion.

  value  : FP64 TFLOP/s at 2n^3 nominal, inputs resident in HBM, device-timed
           with CUDA events (max over ranks).
  e2e    : the same metric through the reference-signature public call
           run_inversion(m, sizes=[256]*64) on a plain (pageable) NumPy array:
           need-ordered H2D, the inversion, D2H into the returned BlockMatrix
           -- all inside the timed region.
  roofline: the dominant kernel K1 (gemm_tma_refill_kernel<4, 64>, FP64 DMMA
           tensor pipe): its algorithmic flops over its own device time (the
           engine's GEMM ops run alone), against the measured DMMA peak
           (MEASURED_PEAKS.json has no FP64 entry).
  cpu_baseline: the reference CPU algorithm (oracle/ port, bitwise equal to
           the reference, profiles/r02_cpu_anchor.jsonl) on a bounded sample of
           the same 64-block structure at n=1024 (rank 0, N=1).
  secondary keys: the opt-in 2n^3 pivot-A schedule on the same matrix, and
           cfg2 (batch of 4 x n=4096, 8 x 512) Eq. 7 / pivot-A.

Multi-GPU (--gpus N, N > 1): one process per GPU (torchrun; started by this
script when it is not already running under torchrun).  The SAME cfg4 matrix
is column-sharded over the N ranks by the level scheduler (home
ranges of 64/N blocks, global levels exchanged over NCCL) -> "scaling":
"strong"; value = 2n^3 / (max over ranks of the step time).

--impl reference: times the reference CPU implementation (the oracle port --
the Python reference cannot travel to the GPU box) on the host cores, same
metric and 64-block structure at n=1024 (bounded sample, n^3 extrapolation to
n=16384 labelled), each step one matrix per host thread.
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

N = 16384
NBLOCKS = 64
METRIC = "FP64 inversion TFLOP/s (2n^3 nominal) and s/inverse, 1/2/4/8 B200 vs CPU ref"
UNIT = "TFLOP/s"
WORKLOAD = ("cfg4: n=16384 float64, N(0,1)/sqrt(n) + 4I (seed 4), 64 diagonal blocks of 256, "
            "run_inversion step engine (Eq. 7, 127 steps)")
CFG2_N, CFG2_NBLOCKS, CFG2_BATCH = 4096, 8, 4
# measured DMMA.8x8x4 chip peak on this pool's B200 (profiles/r01_fp64_dmma_dfma_microbench.txt)
FP64_PEAK_TFLOPS = 36.98
FP64_PEAK_SOURCE = "measured: DMMA.8x8x4 microbench 36.98 TF/s (profiles/r01_fp64_dmma_dfma_microbench.txt); " \
                   "MEASURED_PEAKS.json has no FP64 entry; cuBLAS DGEMM 8192^3 = 35.47 TF/s"


def _driver_fp64_peak():
    """A driver-measured FP64 figure in MEASURED_PEAKS.json (any numeric key with
    'fp64' in its name, TF/s), which then replaces the microbenchmark peak."""
    try:
        peaks = json.loads((Path(__file__).resolve().parent / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return None
    for k, v in peaks.items():
        if "fp64" in k.lower() and isinstance(v, (int, float)) and v > 0:
            return float(v), f"MEASURED_PEAKS.json {k} = {v} (driver-measured)"
    return None


if _driver_fp64_peak() is not None:
    FP64_PEAK_TFLOPS, FP64_PEAK_SOURCE = _driver_fp64_peak()
# CPU sample for the reference arm / cpu_baseline: the same 64-block structure,
# scaled down (n^3 extrapolation to N labelled; anchored by profiles/r02_cpu_anchor.jsonl)
SAMPLE_N = 1024
SAMPLE_SIZES = [16] * 64


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

    g = np.random.default_rng([4, 1000 + seed])
    m = g.standard_normal((SAMPLE_N, SAMPLE_N)) / np.sqrt(SAMPLE_N)
    m[np.diag_indices(SAMPLE_N)] += 4.0
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
    """Sample matrices per step: one per process."""
    return max(1, procs)


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


def _anchor() -> list:
    p = ROOT / "profiles" / "r02_cpu_anchor.jsonl"
    out = []
    if p.exists():
        for ln in p.read_text().splitlines():
            if ln.startswith("{"):
                try:
                    out.append(json.loads(ln))
                except ValueError:
                    pass
    return out


def _cpu_sample(procs: int, min_s: float, max_rounds: int) -> dict:
    """cpu_baseline: rounds of one sample matrix per process (>= min_s of CPU work)."""
    dt, fl, rounds = 0.0, 0.0, 0
    pool = reference_pool(procs)
    try:
        if pool is not None:
            pool.map(_ref_warm, range(procs), chunksize=1)
        while rounds < max_rounds and (rounds == 0 or dt < min_s):
            d1, f1 = reference_sample_step(procs, pool)
            dt, fl, rounds = dt + d1, fl + f1, rounds + 1
    finally:
        if pool is not None:
            pool.close()
    per_inv = dt / (rounds * sample_count(procs)) * procs  # one process's seconds per sample inverse
    return {"value": fl / dt / 1e12, "unit": UNIT, "cores": procs, "kind": "port",
            "sample": f"{rounds} x {sample_count(procs)} matrices n={SAMPLE_N} (64 blocks of {SAMPLE_SIZES[0]}, the "
                      f"cfg4 structure and generator) through the reference run_inversion algorithm (oracle/ port, "
                      f"bitwise equal to the reference), {procs} processes, {dt:.1f} s",
            "s_per_inverse_one_core": per_inv,
            "s_per_inverse_n16384_extrapolated_n3": per_inv * (N / SAMPLE_N) ** 3,
            "anchor": _anchor()}


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    procs = host_threads()
    for _ in range(args.warmup):  # untimed warm-up: tiny problem (imports, page-in)
        _ref_warm(0)
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
    per_inv = total / (args.steps * sample_count(procs)) * procs
    sample = (f"{sample_count(procs)} matrices of n={SAMPLE_N} (64 blocks of {SAMPLE_SIZES[0]}: the cfg4 structure "
              f"and generator, scaled down) per step, reference run_inversion algorithm (oracle/ port, bitwise equal "
              f"to the reference), {procs} processes")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample_n": SAMPLE_N, "sample_blocks": SAMPLE_SIZES[0]},
        "s_per_inverse_one_core": per_inv,
        "s_per_inverse_n16384_extrapolated_n3": per_inv * (N / SAMPLE_N) ** 3,
        "extrapolation_note": "n^3 from the sample; the reference's efficiency grows with n (0.31 GF/s at n=1024, "
                              "0.53 at 2048, 0.55 at cfg2 n=4096 single-threaded: profiles/r02_cpu_anchor.jsonl)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def _load_traffic() -> float | None:
    p = ROOT / "profiles" / "r02_ncu_k1_cfg4.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def _events():
    import torch

    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _time_device(fn, steps: int, warmup: int) -> float:
    """ms per call of fn() (stream-ordered), CUDA events on the current stream."""
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = _events()
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def _secondary_cfg2(bi, steps: int, warmup: int) -> dict:
    """cfg2 (BASELINE configs[1]): batch of 4 x n=4096, 8 x 512, device-resident."""
    from paper_2305_11103_b200.core import _residual_device
    from paper_2305_11103_b200.workloads import cfg2

    ms, sizes = cfg2(CFG2_BATCH, CFG2_N, CFG2_NBLOCKS)
    out = {"workload": "cfg2: batch of 4 x n=4096 float64, N(0,1)/sqrt(n) + 2I, 8 diagonal blocks of 512"}
    for sched in ("eq7", "pivot_a"):
        eng = bi.DeviceEngine(sizes, batch=CFG2_BATCH, schedule=sched)
        eng.load(ms)
        eng.run()
        eng.check()
        fro, _ = _residual_device(eng.M, eng.Minv, batch=True)
        assert np.all(fro <= 1e-9 * CFG2_N), fro
        t = _time_device(eng.run, steps, warmup)
        eng.check()
        out[sched] = {"ms_per_batch": t, "value": CFG2_BATCH * nominal_flops(CFG2_N) / (t * 1e-3) / 1e12,
                      "unit": UNIT, "residual_fro_max": float(np.max(fro))}
        del eng
    bi.release_engines()
    # one cfg2 matrix through the reference-signature call on a NumPy array (e2e)
    import torch

    e2e = []
    for i in range(3 + steps):
        a, b = _events()
        a.record()
        bi.run_inversion(ms[0], sizes=sizes)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            e2e.append(a.elapsed_time(b))
    out["one_matrix_e2e_ms"] = sum(e2e) / len(e2e)
    return out


def run_gpu_arm(args) -> None:
    import torch

    from paper_2305_11103_b200 import build_native

    if build_native.needs_build():
        build_native.build()
    import paper_2305_11103_b200 as bi
    from paper_2305_11103_b200.core import _residual_device
    from paper_2305_11103_b200.workloads import cfg4

    torch.cuda.set_device(0)
    m, sizes = cfg4(N, NBLOCKS)
    stream = torch.cuda.current_stream()

    # ---- headline: cfg4, Eq. 7 step engine, input resident in HBM (2 GiB in + 2 GiB out > L2)
    eng = bi.DeviceEngine(sizes)
    eng.load(m)
    eng.run()  # correctness gate (untimed): residual on the device
    eng.check()
    fro, _ = _residual_device(eng.M, eng.Minv, batch=True)
    assert fro[0] <= 10 * N * np.finfo(float).eps, fro
    for _ in range(args.warmup):
        eng.run()
    torch.cuda.synchronize()
    ev0, ev1 = _events()
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            eng.run()
        ev1.record(stream)
        torch.cuda.synchronize()
    eng.check()
    minv_ref = eng.Minv[0, :, :N].cpu().numpy() if not args.quick else None  # (phase timing overwrites M_inv)
    ms_step = ev0.elapsed_time(ev1) / args.steps
    value = nominal_flops(N) / (ms_step * 1e-3) / 1e12
    counters = eng.counters()
    alg_flops = counters["gemm_flops"] + counters["leaf_flops"]
    launches = eng.launches()

    # ---- per-kernel: the engine's K1 GEMM ops alone and its leaf inversions alone
    reps = max(3, min(args.steps, 10))
    gemm_ms = _time_device(lambda: eng.run_phase(1), reps, 2)
    leaf_ms = _time_device(lambda: eng.run_phase(2), reps, 2)
    k1_tflops = counters["gemm_flops"] / (gemm_ms * 1e-3) / 1e12
    del eng
    bi.release_engines()

    # ---- the opt-in 2n^3 pivot-A schedule on the same matrix
    pa = bi.DeviceEngine(sizes, schedule="pivot_a")
    pa.load(m)
    pa.run()
    pa.check()
    pa_fro, _ = _residual_device(pa.M, pa.Minv, batch=True)
    assert pa_fro[0] <= 10 * N * np.finfo(float).eps, pa_fro
    pa_ms = _time_device(pa.run, args.steps, args.warmup)
    pa.check()
    pa_c = pa.counters()
    pivot_a = {"value": nominal_flops(N) / (pa_ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": pa_ms,
               "algorithmic_tflops": (pa_c["gemm_flops"] + pa_c["leaf_flops"]) / (pa_ms * 1e-3) / 1e12,
               "residual_fro": float(pa_fro[0]),
               "note": "opt-in schedule='pivot_a' (block-level invertor_by_a recursion, 2n^3 flops); "
                       "not the reference's run_inversion step schedule"}
    del pa
    bi.release_engines()

    # ---- e2e: the reference-signature call on a plain NumPy array
    e2e_ms = []
    for i in range(max(1, min(args.warmup, 3)) + args.steps):
        a, b = _events()
        a.record(stream)
        res = bi.run_inversion(m, sizes=sizes)
        b.record(stream)
        torch.cuda.synchronize()
        if i >= max(1, min(args.warmup, 3)):
            e2e_ms.append(a.elapsed_time(b))
    if minv_ref is not None:
        assert np.array_equal(res.store.data, minv_ref)  # the API path computes the same inverse
    del res
    e2e_step = sum(e2e_ms) / len(e2e_ms)
    e2e_value = nominal_flops(N) / (e2e_step * 1e-3) / 1e12
    bi.release_engines()

    cfg2_line = _secondary_cfg2(bi, min(args.steps, 10), args.warmup) if not args.quick else None
    bi.release_engines()

    cpu = None
    if not args.no_cpu_baseline:
        cpu = _cpu_sample(host_threads(), 10.0, 4)

    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n": N, "blocks": f"{NBLOCKS} x {N // NBLOCKS}", "schedule": "eq7",
                   "parallelism": "1 GPU", "l2": "inputs larger than L2 (2 GiB in + 2 GiB out per step)"},
        "s_per_inverse": ms_step * 1e-3,
        "algorithmic_tflops": alg_flops / (ms_step * 1e-3) / 1e12,
        "frac_of_fp64_peak_nominal": value / FP64_PEAK_TFLOPS,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(m.nbytes),
                "d2h_bytes_per_step": int(m.nbytes), "ms_per_step": e2e_step,
                "api": "paper_2305_11103_b200.run_inversion(m, sizes=[256]*64), m a pageable NumPy array"},
        "roofline": {"bound": "tensor", "achieved": k1_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": k1_tflops / FP64_PEAK_TFLOPS, "traffic": _load_traffic(),
                     "kernel": "gemm_tma_refill_kernel<4, 64, Fat> (K1 TMA feeder, engine GEMM ops; 4-warp 64x32 tiles for K >= 1024)",
                     "peak_source": FP64_PEAK_SOURCE,
                     "kernel_ms_per_step": gemm_ms, "kernel_flops_per_step": counters["gemm_flops"],
                     "share_of_step": gemm_ms / ms_step,
                     "leaf_inversion_ms_per_step": leaf_ms,
                     "leaf_inversion_tflops": counters["leaf_flops"] / (leaf_ms * 1e-3) / 1e12},
        "gpu_launches": launches["total"] * args.steps,
        "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
        "residual_fro": float(fro[0]),
        "pivot_a_schedule": pivot_a,
    }
    if cfg2_line is not None:
        line["cfg2_batch"] = cfg2_line
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# multi-GPU: the level scheduler, cfg4 column-sharded over the ranks (strong scaling)
# ---------------------------------------------------------------------------


def run_sharded_arm(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2305_11103_b200 import build_native

    if build_native.needs_build() and int(os.environ.get("LOCAL_RANK", "0")) == 0:
        build_native.build()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BI_BENCH_SHARE_GPU=1 (harness self-test only, never a measurement): ranks
    # share the visible GPUs and exchange over gloo (NCCL refuses two ranks on
    # one GPU), so the N > 1 path can be exercised on a 1-GPU box
    share = os.environ.get("BI_BENCH_SHARE_GPU") == "1"
    if share:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if share:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2305_11103_b200 as bi  # noqa: F401  (after the build on local rank 0)
    from paper_2305_11103_b200.distributed import sharded_engine
    from paper_2305_11103_b200.workloads import cfg4

    m, sizes = cfg4(N, NBLOCKS)
    eng = sharded_engine(sizes)
    eng.load(m)
    eng.run()
    eng.check()
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        eng.run()
    torch.cuda.synchronize()
    ev0, ev1 = _events()
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            eng.run()
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    eng.check()
    t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device="cpu" if share else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = nominal_flops(N) / (ms_step * 1e-3) / 1e12
    # e2e: host matrix in (each rank its column slab), inverse gathered to rank 0's host memory
    e2e = []
    for i in range(1 + args.steps):
        dist.barrier()
        a, b = _events()
        a.record(stream)
        eng.load(m)
        eng.run()
        eng.check()
        full = eng.gather(0)
        b.record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device="cpu" if share else "cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        if i:
            e2e.append(float(tt.item()))
    if rank == 0:
        fro = bi.residual_frobenius(m, full)
        assert fro <= 10 * N * np.finfo(float).eps, fro
        e2e_step = sum(e2e) / len(e2e)
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": N, "blocks": f"{NBLOCKS} x {N // NBLOCKS}", "schedule": "eq7",
                       "parallelism": f"column-sharded level scheduler over {world} ranks (SURVEY 8e)",
                       "l2": "inputs larger than L2"},
            "s_per_inverse": ms_step * 1e-3,
            "frac_of_fp64_peak_nominal": value / (world * FP64_PEAK_TFLOPS),
            "e2e": {"value": nominal_flops(N) / (e2e_step * 1e-3) / 1e12, "unit": UNIT,
                    "h2d_bytes_per_step": int(m.nbytes), "d2h_bytes_per_step": int(m.nbytes),
                    "ms_per_step": e2e_step, "api": "sharded engine load (host) + run + gather to rank 0"},
            "gpu_launches": (eng.launches() * args.steps) if eng.launches() is not None else None,
            "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
            "residual_fro": float(fro),
        }
        # K1's algorithmic flops per GPU (arrows 2n^3 - 2n^2 b, up/down n^3 - n^2 b) over the WHOLE
        # sharded step -- leaf steps and exchanges included, so a lower bound of the kernel's own rate
        b = N // NBLOCKS
        gemm_flops = 3.0 * N**3 - 3.0 * N**2 * b
        ach = gemm_flops / world / (ms_step * 1e-3) / 1e12
        line["roofline"] = {"bound": "tensor", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": UNIT,
                            "frac": ach / FP64_PEAK_TFLOPS, "traffic": None, "peak_source": FP64_PEAK_SOURCE,
                            "kernel": "gemm_tma_refill_kernel (K1, engine GEMM ops), per GPU",
                            "note": "per-GPU algorithmic GEMM flops over the whole sharded step (leaves and "
                                    "exchanges included): a lower bound of the kernel's own rate"}
        if share:
            line["harness_self_test"] = "BI_BENCH_SHARE_GPU=1: ranks share one GPU over gloo -- not a measurement"
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _self_launch(args, argv) -> int:
    """--gpus N > 1 outside torchrun: start N ranks with torch.distributed.run."""
    import socket

    import torch

    visible = torch.cuda.device_count()
    if visible < args.gpus and os.environ.get("BI_BENCH_SHARE_GPU") != "1":
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {visible}", file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def main(argv=None) -> None:
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip the cfg2 secondary keys and the e2e equality check")
    args = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if world != args.gpus:
        if world == 1 and "RANK" not in os.environ and args.gpus > 1:
            sys.exit(_self_launch(args, argv))
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if world > 1:
        run_sharded_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
