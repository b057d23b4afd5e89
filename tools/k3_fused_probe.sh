# K3 knobs A/B: bitwise checkers (fast path, fused kernel), then graph-replay times.
python tools/k3_fast_check.py BI_GJ_FAST 2>&1 | tail -1
python tools/k3_fast_check.py BI_GJ_FUSED 2>&1 | tail -1
BI_GJ_FAST_SMALL=0 python tools/k3_fast_check.py BI_GJ_FUSED 2>&1 | tail -1
for spec in "64 256" "8 512" "32 512"; do
  set -- $spec
  for env in "BI_GJ_FAST_SMALL=0 BI_GJ_FUSED=0" "BI_GJ_FAST_SMALL=1 BI_GJ_FUSED=0" "BI_GJ_FAST_SMALL=1 BI_GJ_FUSED=1"; do
    echo -n "[$env] "; env $env timeout 120 python tools/profile_inv_graph.py --count $1 --n $2
  done
done
