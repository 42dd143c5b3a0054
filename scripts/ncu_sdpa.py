"""ncu target: torch SDPA (cuDNN/flash backend) at C2, for comparison with attn_kernel."""
import torch
B, H, S, D = 8, 32, 2048, 128
q = torch.randn(B, H, S, D, device="cuda").bfloat16(); k = torch.randn(B, H, S, D, device="cuda").bfloat16()
v = torch.randn(B, H, S, D, device="cuda").bfloat16()
for _ in range(3):
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
print("done")
