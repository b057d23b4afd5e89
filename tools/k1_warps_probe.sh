# K1 warp-tile A/B (BI_GEMM_WARPS 8 / 4 / auto): GEMM correctness, engine device times.
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -m gpu -k "gemm" 2>&1 | tail -1
for w in 8 auto 8 auto; do echo "== BI_GEMM_WARPS=$w"; if [ $w = auto ]; then timeout 300 python tools/engine_time.py; else BI_GEMM_WARPS=$w timeout 300 python tools/engine_time.py; fi; done
