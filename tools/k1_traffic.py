"""DRAM traffic of K1 on the bench workload (for bench.py's roofline.traffic).

  run:        python tools/k1_traffic.py run
              -- one engine K1 phase (cfg2, batch 4) after one warm run; wrap
                 in ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
                 gpu__time_duration.sum --nvtx --nvtx-include k1_phase/
  summarize:  python tools/k1_traffic.py summarize <ncu.csv> <out.json>
              -- per-launch DRAM bytes (read + write) vs the engine's
                 algorithmic GEMM bytes (bi_engine_counters out[5])
"""

import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

BATCH, SIZES = 4, [512] * 8


def run():
    import torch

    import paper_2305_11103_b200 as bi
    from paper_2305_11103_b200 import workloads

    ms, _ = workloads.cfg2(batch=BATCH)
    eng = bi.DeviceEngine(SIZES, BATCH)
    eng.load(ms)
    eng.run_phase(1)  # warm (outside the NVTX range ncu filters on)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("k1_phase")
    eng.run_phase(1)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("engine launches:", eng.launches())


def summarize(csv_path, out_path):
    per = defaultdict(dict)
    names = {}
    with open(csv_path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        i = int(row["ID"])
        names[i] = row["Kernel Name"]
        v = float(row["Metric Value"].replace(",", ""))
        unit = row["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}[unit]
        per[i][row["Metric Name"]] = v * scale
    ids = sorted(per)
    rd = sum(per[i].get("dram__bytes_read.sum", 0) for i in ids)
    wr = sum(per[i].get("dram__bytes_write.sum", 0) for i in ids)
    t = sum(per[i].get("gpu__time_duration.sum", 0) for i in ids)
    c = _counters()
    n = len(ids)
    out = {
        "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                  "--clock-control none, one engine K1 phase (run_phase mask 1) of the bench workload "
                  "(cfg2: batch 4 x n=4096, 8 x 512 blocks)",
        "kernels": sorted(set(names.values())),
        "launches": n,
        "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_launch": (rd + wr) / n,
        "algorithmic_bytes_per_step": c["gemm_bytes"],
        "algorithmic_bytes_per_launch": c["gemm_bytes"] / n,
        "traffic_over_algorithmic": (rd + wr) / c["gemm_bytes"],
        "gemm_flops_per_step": c["gemm_flops"],
        "ncu_kernel_time_s_cold_serialised": t,
        "ncu_tflops_cold_serialised": c["gemm_flops"] / t / 1e12 if t else None,
    }
    Path(out_path).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


def _counters():
    import ctypes

    from paper_2305_11103_b200 import _lib

    lib = _lib.lib()
    h = _lib._vp()
    arr = (_lib._c_i64 * len(SIZES))(*SIZES)
    assert lib.bi_engine_create(ctypes.byref(h), len(SIZES), arr, BATCH) == 0
    out = (ctypes.c_double * 6)()
    assert lib.bi_engine_counters(h, 1, 2 * len(SIZES) - 1, out) == 0
    lib.bi_engine_destroy(h)
    return {"gemm_flops": out[3], "gemm_bytes": out[5]}


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        summarize(sys.argv[2], sys.argv[3])
