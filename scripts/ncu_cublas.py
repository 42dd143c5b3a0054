"""ncu target: the cuBLAS GEMM of the C4 shape (X[65536, 4096] @ Yt^T), for comparison with K2."""
import torch
X = torch.randn(65536, 4096, device="cuda").bfloat16(); Yt = torch.randn(4096, 4096, device="cuda").bfloat16()
for _ in range(3):
    o = X @ Yt.T
torch.cuda.synchronize()
print("done")
