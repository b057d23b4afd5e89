# Sub-panel lookahead (BI_GJ_SUBLA) vs the chain: bitwise, engine tests, graph-replay and engine times.
python tools/k3_fast_check.py BI_GJ_SUBLA 2>&1 | tail -8
BI_GJ_SUBLA=1 timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py -q -x -m gpu 2>&1 | tail -1
for spec in "64 256" "8 512" "32 512"; do set -- $spec
  for v in 0 1; do echo -n "[BI_GJ_SUBLA=$v] "; BI_GJ_SUBLA=$v timeout 120 python tools/profile_inv_graph.py --count $1 --n $2; done
done
for v in 0 1 0 1; do echo -n "[BI_GJ_SUBLA=$v] "; BI_GJ_SUBLA=$v timeout 300 python tools/engine_time.py | tr '\n' ' '; echo; done
