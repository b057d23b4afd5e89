"""cuBLAS DGEMM ceiling via torch.matmul(float64) -- test/measurement only."""
import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10 if n < 8192 else 5
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cublas dgemm n={n}: {2*n**3/ms/1e9:.2f} TFLOP/s ({ms:.3f} ms)")
for n in (512, 1024, 4096):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda") + n * torch.eye(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        x = torch.linalg.inv(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        x = torch.linalg.inv(a)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"torch.linalg.inv (cuSOLVER) n={n}: {ms:.3f} ms, {2*n**3/ms/1e9:.2f} TFLOP/s nominal")
