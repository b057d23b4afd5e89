# K3 leaf-step probe (GPU box): one engine ◇ step's shapes timed from a CUDA graph
# under the K3 knobs, and the cfg4 / cfg2 engines with and without leaves.
for spec in "64 256" "8 512" "32 512"; do
  set -- $spec
  for env in "" "BI_GJ_WINDOW=256" "BI_GJ_NB=16" "BI_GJ_FAST=0" "BI_PDL=0"; do
    echo -n "[$env] "; env $env python tools/profile_inv_graph.py --count $1 --n $2
  done
done
python - <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
import paper_2305_11103_b200 as bi
from paper_2305_11103_b200.workloads import cfg4
m, sizes = cfg4()
eng = bi.DeviceEngine(sizes, batch=1)
eng.load(m[None])
for _ in range(2): eng.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): eng.run()
e1.record(); torch.cuda.synchronize()
print("cfg4 skip_leaves", os.environ.get("BI_DEBUG_SKIP_LEAVES", "0"), "ms", e0.elapsed_time(e1) / 3)
PY
