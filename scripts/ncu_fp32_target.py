"""Minimal launcher for ncu captures of the fp32 modes at the C2 (attention) and C3 (FFN) shapes."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_07829_b200 import ops

what = sys.argv[1] if len(sys.argv) > 1 else "attn"
g = torch.Generator(device="cuda").manual_seed(0)
r = lambda *s: torch.randn(*s, device="cuda", generator=g)  # noqa: E731
if what == "attn":
    Q, K, Vt = r(256, 2048, 128), r(256, 2048, 128), r(256, 128, 2048)
    fn = lambda: ops.attention(Q, K, Vt)  # noqa: E731
else:
    M, D, F = 8192, 4096, 14336
    X, Wt, Vt, Ut = r(M, D), r(F, D) * D ** -0.5, r(F, D) * D ** -0.5, r(D, F) * F ** -0.5
    fn = lambda: ops.rms_ffn_swiglu(X, Wt, Vt, Ut)  # noqa: E731
for _ in range(3):
    fn()
torch.cuda.synchronize()
print("done", what)
