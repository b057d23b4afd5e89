"""One cuBLAS DGEMM shape for ncu (measurement only): python cublas_one.py M N K BATCH"""
import sys
import torch

m, n, k, b = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (8192, 8192, 8192, 1)
a = torch.randn(b, m, k, dtype=torch.float64, device="cuda")
bb = torch.randn(b, k, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = torch.bmm(a, bb)
torch.cuda.synchronize()
