# cfg2 batch (4 lanes) with the fused single-launch K3 and lane skews / priority modes.
for env in "BI_GJ_FUSED=0" "BI_GJ_FUSED=1" "BI_GJ_FUSED=1 BI_ENGINE_SKEW=1" "BI_GJ_FUSED=1 BI_ENGINE_SKEW=2" \
           "BI_GJ_FUSED=1 BI_PRIORITY_MODE=1" "BI_GJ_FUSED=1 BI_PRIORITY_MODE=4 BI_ENGINE_SKEW=1" \
           "BI_GJ_FUSED=0 BI_ENGINE_SKEW=1" "BI_GJ_FUSED=1 BI_PRIORITY_MODE=0"; do
  echo -n "[$env] "; env $env timeout 200 python tools/engine_time.py cfg2 --reps 5
done
