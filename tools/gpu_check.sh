BI_GEMM_TMA=0 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x 2>&1 | tail -1
BI_GEMM_TMA=0 BI_GEMM_CP_TN=128 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x 2>&1 | tail -1
for tn in 128 64 128 64; do echo "cp.async TN $tn"; BI_GEMM_TMA=0 BI_GEMM_CP_TN=$tn python tools/gemm_sweep.py 2>&1 | sed -n '1,6p'; done
