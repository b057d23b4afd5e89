"""Where one cfg2 matrix's end-to-end time goes (n=4096, 8 x 512):
device-resident engine run, run_host with page-locked in/out, run_host with
a pageable input (the engine's need-ordered staging) and page-locked output,
and the public run_inversion(m, sizes) call.  CUDA events, warm, 10 reps."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_11103_b200 as bi  # noqa: E402
from paper_2305_11103_b200.workloads import cfg2, cfg4  # noqa: E402


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for name, (m, sizes) in (("cfg2 one matrix", (cfg2(1)[0][0], cfg2(1)[1])), ("cfg4", cfg4())):
    reps = 10 if m.shape[0] <= 4096 else 3
    eng = bi.DeviceEngine(sizes)
    eng.load(m)
    t_dev = timed(eng.run, reps)
    pin_in = torch.from_numpy(m).pin_memory().numpy()
    pin_out = torch.empty(m.shape, dtype=torch.float64, pin_memory=True).numpy()
    t_pp = timed(lambda: (eng.run_host(pin_in, pin_out), eng.check()), reps)
    t_gp = timed(lambda: (eng.run_host(m, pin_out), eng.check()), reps)
    out_np = np.empty_like(m)
    t_gg = timed(lambda: (eng.run_host(m, out_np), eng.check()), reps)
    del eng
    t_api = timed(lambda: bi.run_inversion(m, sizes=sizes), reps)
    bi.release_engines()
    print(f"{name}: device {t_dev:.2f} ms | run_host pinned/pinned {t_pp:.2f} | pageable in/pinned out {t_gp:.2f} "
          f"| pageable/pageable {t_gg:.2f} | run_inversion(m) {t_api:.2f} ms", flush=True)
