"""Probe: vendor FP64 yardsticks on the B200 (context only, never shipped):
cuBLAS DGEMM 8192^3 (torch.matmul float64) and cuSOLVER potrf (torch.linalg.cholesky)."""
import torch, time
d = torch.device("cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=d); b = torch.randn(n, n, dtype=torch.float64, device=d)
    ms = t(lambda: torch.matmul(a, b))
    print(f"cublas dgemm {n}^3: {2*n**3/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms)")
for n in (8192, 16384, 32768):
    m = torch.randn(n, n, dtype=torch.float64, device=d)
    a = m @ m.T + n * torch.eye(n, dtype=torch.float64, device=d)
    del m
    ms = t(lambda: torch.linalg.cholesky(a), reps=3)
    print(f"cusolver potrf n={n}: {n**3/3/ms/1e9:.2f} TFLOP/s ({ms:.1f} ms)")
    del a
