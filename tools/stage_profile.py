"""Timing of the page-locked staging helpers (_lib.to_device / download / _threaded_copy) at 128 MiB."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2305_11103_b200 as bi
from paper_2305_11103_b200 import _lib
n = 4096
x = np.random.default_rng(1).standard_normal((n, n))
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d = _lib.to_device(x); torch.cuda.synchronize(); t1 = time.perf_counter()
    out = np.empty_like(x); _lib.download(d, out); t2 = time.perf_counter()
    pin = torch.empty(x.shape, dtype=torch.float64, pin_memory=True).numpy(); t3 = time.perf_counter(); _lib._threaded_copy(pin, x); t4 = time.perf_counter()
    np.copyto(pin, x); t5 = time.perf_counter()
print(f"upload {1e3*(t1-t0):.1f} ms, download {1e3*(t2-t1):.1f} ms, threaded copy 128 MiB {1e3*(t4-t3):.1f} ms, single copy {1e3*(t5-t4):.1f} ms, cpus {__import__('os').cpu_count()}")
