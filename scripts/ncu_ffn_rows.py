"""ncu target: the default K1 fused launch at a given row count (Llama-3-8B weights), n times."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_07829_b200 import ops

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
D, F = 4096, 14336
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(M, D, device="cuda", generator=g).bfloat16()
Wt = (torch.randn(F, D, device="cuda", generator=g) * D ** -0.5).bfloat16()
Vt = (torch.randn(F, D, device="cuda", generator=g) * D ** -0.5).bfloat16()
Ut = (torch.randn(D, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
for _ in range(n):
    ops.rms_ffn_swiglu(X, Wt, Vt, Ut)
torch.cuda.synchronize()
print("done", M)
