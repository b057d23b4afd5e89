# Engine GEMM launches with / without programmatic dependent launch.
for v in 0 1 0 1; do echo "== BI_ENGINE_PDL=$v"; BI_ENGINE_PDL=$v timeout 300 python tools/engine_time.py; done
BI_ENGINE_PDL=1 timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -m gpu 2>&1 | tail -1
