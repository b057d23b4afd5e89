"""Where the first cfg4 call goes: engine bind, load, graph capture, staging allocation."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2305_11103_b200 as bi
from paper_2305_11103_b200.workloads import cfg4
m, sizes = cfg4()
torch.cuda.init(); torch.cuda.synchronize()
t0 = time.perf_counter(); eng = bi.DeviceEngine(sizes); torch.cuda.synchronize(); t1 = time.perf_counter()
eng.load(m[None]); torch.cuda.synchronize(); t2 = time.perf_counter()
eng.run(); torch.cuda.synchronize(); t3 = time.perf_counter()
eng.run(); torch.cuda.synchronize(); t4 = time.perf_counter()
out = torch.empty(m.shape, dtype=torch.float64, pin_memory=True).numpy(); t5 = time.perf_counter()
eng.run_host(m[None], out[None]); torch.cuda.synchronize(); t6 = time.perf_counter()
eng.run_host(m[None], out[None]); torch.cuda.synchronize(); t7 = time.perf_counter()
print(f"bind {1e3*(t1-t0):.0f} ms, load {1e3*(t2-t1):.0f}, first run (capture) {1e3*(t3-t2):.0f}, warm run {1e3*(t4-t3):.0f}, pinned out alloc {1e3*(t5-t4):.0f}, first run_host {1e3*(t6-t5):.0f}, warm run_host {1e3*(t7-t6):.0f}")
