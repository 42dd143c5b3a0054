"""ncu DRAM bytes of the torch/cuBLAS unfused FFN at the Llama-3-70B shape (C5), one step."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
M, D, F = 32768, 8192, 28672
X = torch.randn(M, D, device="cuda").bfloat16()
Wt = (torch.randn(F, D, device="cuda") * D ** -0.5).bfloat16(); Vt = (torch.randn(F, D, device="cuda") * D ** -0.5).bfloat16()
Ut = (torch.randn(D, F, device="cuda") * F ** -0.5).bfloat16()
def step():
    Xn = (X.float() * torch.rsqrt(X.float().square().mean(-1, keepdim=True))).bfloat16()
    return (torch.nn.functional.silu(Xn @ Wt.T) * (Xn @ Vt.T)) @ Ut.T
step(); torch.cuda.synchronize()
torch.cuda.profiler.start(); step(); torch.cuda.synchronize(); torch.cuda.profiler.stop()
