"""Host-side facts of the GPU box that size the full-size tests and the e2e
path: cores, RAM, LAPACK speed at n=16384, NumPy normal-draw rate, and the
host<->device copy options for a pageable 2 GiB NumPy array (pageable
cudaMemcpy, staged through page-locked memory, cudaHostRegister).
    python tools/host_probe.py
"""

from __future__ import annotations

import json
import os
import time

import numpy as np


def main() -> None:
    import torch

    out = {"threads": len(os.sched_getaffinity(0))}
    with open("/proc/meminfo") as f:
        for ln in f:
            if ln.startswith(("MemTotal", "MemAvailable")):
                out[ln.split(":")[0]] = ln.split()[1] + " kB"
    with open("/sys/kernel/mm/transparent_hugepage/enabled") as f:
        out["thp"] = f.read().strip()
    g = np.random.default_rng(5)
    t = time.perf_counter()
    a = g.standard_normal((4096, 65536))
    out["normal_draw_Mps"] = a.size / (time.perf_counter() - t) / 1e6
    n = 1 << 14
    m = np.random.default_rng(4).standard_normal((n, n)) / 128.0
    m[np.diag_indices(n)] += 4.0
    # first touch of a fresh 2 GiB array
    t = time.perf_counter()
    e = np.empty((n, n))
    e.fill(0.0)
    out["first_touch_2GiB_s"] = time.perf_counter() - t
    dev = torch.empty((n, n), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(2):
        t = time.perf_counter()
        dev.copy_(torch.from_numpy(m))
        torch.cuda.synchronize()
        out["pageable_h2d_GBps"] = m.nbytes / (time.perf_counter() - t) / 1e9
    for _ in range(2):
        t = time.perf_counter()
        e2 = dev.cpu().numpy()
        out["pageable_d2h_new_GBps"] = m.nbytes / (time.perf_counter() - t) / 1e9
    pin = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    t = time.perf_counter()
    torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    out["pinned_alloc_2GiB_s"] = time.perf_counter() - t
    pn = pin.numpy()
    for th in (1, 4, 8, 16):
        from concurrent.futures import ThreadPoolExecutor

        flat_d, flat_s = pn.reshape(-1), m.reshape(-1)
        b = [flat_d.size * i // th for i in range(th + 1)]
        with ThreadPoolExecutor(th) as ex:
            t = time.perf_counter()
            list(ex.map(lambda i: np.copyto(flat_d[b[i]:b[i + 1]], flat_s[b[i]:b[i + 1]]), range(th)))
            out[f"memcpy_to_pinned_{th}thr_GBps"] = m.nbytes / (time.perf_counter() - t) / 1e9
    cudart = torch.cuda.cudart()
    t = time.perf_counter()
    rc = cudart.cudaHostRegister(m.ctypes.data, m.nbytes, 0)
    out["hostregister_2GiB_s"] = time.perf_counter() - t
    out["hostregister_rc"] = int(rc)
    t = time.perf_counter()
    dev.copy_(torch.from_numpy(m))
    torch.cuda.synchronize()
    out["registered_h2d_GBps"] = m.nbytes / (time.perf_counter() - t) / 1e9
    t = time.perf_counter()
    cudart.cudaHostUnregister(m.ctypes.data)
    out["hostunregister_s"] = time.perf_counter() - t
    del e2
    t = time.perf_counter()
    inv = np.linalg.inv(m)
    out["lapack_inv_n16384_s"] = time.perf_counter() - t
    out["lapack_inv_GFps"] = 2 * n ** 3 / out["lapack_inv_n16384_s"] / 1e9
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
