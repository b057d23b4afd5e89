python tools/k3_fast_check.py BI_GJ_FUSED 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -x -m gpu 2>&1 | tail -1
for spec in "64 256" "8 512" "32 512" "1 5000"; do set -- $spec; timeout 120 python tools/profile_inv_graph.py --count $1 --n $2; done
timeout 300 python tools/engine_time.py
