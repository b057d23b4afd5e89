import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2305_11103_b200 import _lib
from paper_2305_11103_b200.core import device_inverse, _residual_device
from paper_2305_11103_b200.recursive import inplace_by_a_device
from paper_2305_11103_b200.workloads import cfg3
m, split = cfg3()
D = m[split:, split:].copy()
dD = _lib.to_device(D)
for leaf in (256, 512, 1024):
    x = dD.clone()
    inplace_by_a_device(x, leaf); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x = dD.clone(); e0.record(); inplace_by_a_device(x, leaf); e1.record(); torch.cuda.synchronize()
    rf, rm = _residual_device(dD, x)
    print(f"inplace_by_a 5000 leaf {leaf}: {e0.elapsed_time(e1):.2f} ms, residual_F {rf[0]:.2e}")
out = _lib.empty_matrix(5000, 5000)
device_inverse(dD, out); torch.cuda.synchronize()
e0.record(); device_inverse(dD, out); e1.record(); torch.cuda.synchronize()
rf, rm = _residual_device(dD, out)
print(f"K3 5000: {e0.elapsed_time(e1):.2f} ms, residual_F {rf[0]:.2e}")
