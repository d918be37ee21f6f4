"""Probe target: one cuBLAS DGEMM 8192^3 (torch.matmul float64) after a warm-up, for ncu."""
import torch
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
torch.matmul(a, b)
torch.cuda.synchronize()
torch.matmul(a, b)
torch.cuda.synchronize()
