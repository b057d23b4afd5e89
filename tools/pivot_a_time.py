"""Device time of the opt-in pivot-A schedule on cfg4 and the cfg2 batch."""
import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2305_11103_b200 as bi
from paper_2305_11103_b200.workloads import cfg4, cfg2
for name, (ms, sizes) in (("cfg4", (cfg4()[0][None], cfg4()[1])), ("cfg2", cfg2(4))):
    eng = bi.DeviceEngine(sizes, batch=ms.shape[0], schedule="pivot_a"); eng.load(ms)
    for _ in range(2): eng.run()
    torch.cuda.synchronize(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): eng.run()
    b.record(); torch.cuda.synchronize(); print(f"pivot_a {name}: {a.elapsed_time(b)/3:.2f} ms")
