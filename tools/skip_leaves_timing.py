import os, sys, torch
sys.path.insert(0, '.')
import paper_2305_11103_b200 as bi
from paper_2305_11103_b200.workloads import cfg2
ms, sizes = cfg2(4)
eng = bi.DeviceEngine(sizes, batch=4)
eng.load(ms)
for _ in range(3): eng.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): eng.run()
e1.record(); torch.cuda.synchronize()
print(os.environ.get("BI_DEBUG_SKIP_LEAVES", "0"), os.environ.get("BI_ENGINE_LANES", "-"), "ms per batch", e0.elapsed_time(e1) / 5)
