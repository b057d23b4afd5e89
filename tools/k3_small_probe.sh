# Single-CTA fast panels (BI_GJ_FAST_SMALL) A/B: bitwise checker, then graph-replay times.
python tools/k3_fast_check.py 2>&1 | tail -15
for spec in "64 256" "8 512" "32 512"; do
  set -- $spec
  for env in "BI_GJ_FAST_SMALL=0" "BI_GJ_FAST_SMALL=1"; do
    echo -n "[$env] "; env $env python tools/profile_inv_graph.py --count $1 --n $2
  done
done
