import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_2305_11103_b200 as bi
from paper_2305_11103_b200.workloads import cfg2
ms, sizes = cfg2(1); m = ms[0]
eng = bi.DeviceEngine(sizes)
pin_out = torch.empty(m.shape, dtype=torch.float64, pin_memory=True).numpy()
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.run_host(m, pin_out); eng.check()
    print(f"call {i}: {1e3*(time.perf_counter()-t0):.2f} ms wall", file=sys.stderr, flush=True)
