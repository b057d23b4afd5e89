# K1 tile A/B: 64 x 64 (3 CTAs/SM) vs 128 x 64; correctness + bitwise, sweep, engine.
timeout 900 python -m pytest tests/test_gpu_knobs.py -q -x -m gpu -k "bitwise and not fused" 2>&1 | tail -1
BI_GEMM_TM=64 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -m gpu -k "gemm" 2>&1 | tail -1
for tm in 128 64; do echo "== BI_GEMM_TM=$tm"; BI_GEMM_TM=$tm timeout 300 python tools/gemm_sweep.py 2>&1 | head -14; done
for tm in 128 64 auto; do echo "== BI_GEMM_TM=$tm"; if [ $tm = auto ]; then timeout 300 python tools/engine_time.py; else BI_GEMM_TM=$tm timeout 300 python tools/engine_time.py; fi; done
for k in 1024 2048; do echo "== auto, BI_GEMM_TM64_K=$k"; BI_GEMM_TM64_K=$k timeout 300 python tools/engine_time.py; done
