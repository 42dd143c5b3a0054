import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_07829_b200 import ops
def cmp(a, b, name):
    d = (a.float() - b.float()).abs()
    n = (a != b).sum().item()
    idx = (a != b).nonzero()[:5].tolist()
    print(f"{name}: {n} differ / {a.numel()}, max diff {d.max().item():.4g}, first {idx}", flush=True)
g = torch.Generator(device="cuda").manual_seed(1)
M, D, F = 4096, 1024, 2816
X = torch.randn(M, D, device="cuda", generator=g).bfloat16()
Wt, Vt = (torch.randn(F, D, device="cuda", generator=g).mul(0.03).bfloat16() for _ in range(2))
Ut = torch.randn(D, F, device="cuda", generator=g).mul(0.02).bfloat16()
a = ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule="two_phase").clone()
a2 = ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule="two_phase").clone()
b = ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule="fused").clone()
b2 = ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule="fused").clone()
c = ops.rms_ffn_swiglu(X * 2, Wt, Vt, Ut, schedule="two_phase").clone()
torch.cuda.synchronize()
cmp(a, a2, "two_phase repeat"); cmp(b, b2, "fused repeat"); cmp(a, b, "two_phase vs fused"); cmp(a, c, "O(2X) vs O(X) two_phase")
X = torch.randn(8192, 4096, device="cuda", generator=g).bfloat16(); Yt = torch.randn(4096, 4096, device="cuda", generator=g).bfloat16()
o1 = ops.layernorm_matmul(X, Yt).clone(); o2 = ops.layernorm_matmul(X, Yt).clone(); o3 = ops.layernorm_matmul(X * 2, Yt).clone()
torch.cuda.synchronize()
cmp(o1, o2, "K2 repeat"); cmp(o1, o3, "K2 O(2X) vs O(X)")
