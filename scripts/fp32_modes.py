"""fp32-in/fp32-out modes at the C2/C3/C4 shapes: device time and TFLOP/s (CUDA events, 3 warm-up + 5 timed)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_07829_b200 import ops


def t(fn, n=5, w=3):
    for _ in range(w):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


g = torch.Generator(device="cuda").manual_seed(0)
r = lambda *s: torch.randn(*s, device="cuda", generator=g)  # noqa: E731
M, D, F = 8192, 4096, 14336
X, Wt, Vt, Ut = r(M, D), r(F, D) * D ** -0.5, r(F, D) * D ** -0.5, r(D, F) * F ** -0.5
ms = t(lambda: ops.rms_ffn_swiglu(X, Wt, Vt, Ut))
print(f"K1 fp32 C3: {ms:.2f} ms {6 * M * D * F / ms / 1e9:.1f} TFLOP/s")
rows = torch.arange(0, M, 97, device="cuda")
Xr = X[rows].double()
Xn = Xr * torch.rsqrt(Xr.pow(2).mean(-1, keepdim=True))
a, b = Xn @ Wt.double().T, Xn @ Vt.double().T
ref = (a * torch.sigmoid(a) * b) @ Ut.double().T
O = ops.rms_ffn_swiglu(X, Wt, Vt, Ut)[rows].double()
print(f"K1 fp32 C3 {rows.numel()} rows: max|d|/max|ref| = {float((O - ref).abs().max() / ref.abs().max()):.2e}")
del X, Wt, Vt, Ut
X, Yt = r(65536, 4096), r(4096, 4096)
ms = t(lambda: ops.layernorm_matmul(X, Yt))
print(f"K2 fp32 C4: {ms:.2f} ms {2 * 65536 * 4096 * 4096 / ms / 1e9:.1f} TFLOP/s")
rows = torch.arange(0, 65536, 811, device="cuda")
Xr = X[rows].double()
ref = ((Xr - Xr.mean(-1, keepdim=True)) / Xr.std(-1, unbiased=False, keepdim=True)) @ Yt.double().T
O = ops.layernorm_matmul(X, Yt)[rows].double()
print(f"K2 fp32 C4 {rows.numel()} rows: max|d|/max|ref| = {float((O - ref).abs().max() / ref.abs().max()):.2e}")
del X, Yt
Q, K, V = r(256, 2048, 128), r(256, 2048, 128), r(256, 128, 2048)
ms = t(lambda: ops.attention(Q, K, V))
print(f"K3 fp32 C2: {ms:.2f} ms {4 * 256 * 2048 * 2048 * 128 / ms / 1e9:.1f} TFLOP/s")
ref = torch.softmax((Q[:8] @ K[:8].transpose(1, 2)).double() / 128 ** 0.5, -1) @ V[:8].transpose(1, 2).double()
O = ops.attention(Q, K, V)[:8].double()
print(f"K3 fp32 C2 heads 0-7: max|d|/max|ref| = {float((O - ref).abs().max() / ref.abs().max()):.2e}")
