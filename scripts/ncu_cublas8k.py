"""ncu target: cuBLAS bf16 8192^3 (MEASURED_PEAKS' GEMM) and the C3 gate GEMM shape, for comparison with K1."""
import torch
a = torch.randn(8192, 8192, device="cuda").bfloat16(); b = torch.randn(8192, 8192, device="cuda").bfloat16()
x = torch.randn(8192, 4096, device="cuda").bfloat16(); w = torch.randn(28672, 4096, device="cuda").bfloat16()
for _ in range(3):
    c = a @ b
    h = x @ w.T
torch.cuda.synchronize()
print("done")
