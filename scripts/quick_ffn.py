"""Scratch: K1 correctness at small shapes vs torch fp32 and timing at the 8B shape."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_07829_b200 import ops

def ref(X, Wt, Vt, Ut, eps=0.0):
    X, Wt, Vt, Ut = (t.float() for t in (X, Wt, Vt, Ut))
    r = torch.rsqrt((X * X).mean(1, keepdim=True) + eps)
    g = (X @ Wt.T) * r
    u = (X @ Vt.T) * r
    h = (g * torch.sigmoid(g) * u).bfloat16().float()
    return h @ Ut.T

def check(M, D, F, N, sched, scale=0.05):
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn(M, D, device="cuda", generator=g).bfloat16()
    Wt = (torch.randn(F, D, device="cuda", generator=g) * scale).bfloat16()
    Vt = (torch.randn(F, D, device="cuda", generator=g) * scale).bfloat16()
    Ut = (torch.randn(N, F, device="cuda", generator=g) * scale).bfloat16()
    O = ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule=sched)
    torch.cuda.synchronize()
    R = ref(X, Wt, Vt, Ut)
    err = (O.float() - R).abs().max().item() / R.abs().max().item()
    print(f"M={M} D={D} F={F} N={N} {sched}: max|d|/max|ref| = {err:.3e}", flush=True)
    return err

for shape in [(128, 64, 128, 256), (300, 200, 136, 264), (1024, 512, 1024, 512), (2048, 256, 512, 256), (4096, 512, 2048, 512), (8192, 1024, 4096, 1024)]:
    for s in ("two_phase", "fused"):
        check(*shape, s)

M, D, F = 8192, 4096, 14336
X = torch.randn(M, D, device="cuda").bfloat16()
Wt = (torch.randn(F, D, device="cuda") * 0.02).bfloat16()
Vt = (torch.randn(F, D, device="cuda") * 0.02).bfloat16()
Ut = (torch.randn(D, F, device="cuda") * 0.02).bfloat16()
flops = 6 * M * D * F
for s in ("two_phase", "fused"):
    for _ in range(3):
        O = ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 10
    e0.record()
    for _ in range(n):
        ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule=s, out=O)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{s}: {ms:.3f} ms  {flops/ms/1e9:.1f} TFLOP/s", flush=True)
    R = ref(X[:256], Wt, Vt, Ut)
    print(f"  8B rows 0..255 err {(O[:256].float()-R).abs().max().item()/R.abs().max().item():.3e}")
# torch unfused reference timing
def unfused(X, Wt, Vt, Ut):
    r = torch.rsqrt((X.float()**2).mean(1, keepdim=True))
    xn = (X.float() * r).bfloat16()
    g = xn @ Wt.T; u = xn @ Vt.T
    return (torch.nn.functional.silu(g) * u) @ Ut.T
for _ in range(3): unfused(X, Wt, Vt, Ut)
torch.cuda.synchronize()
e0.record()
for _ in range(10): unfused(X, Wt, Vt, Ut)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)/10
print(f"torch unfused (cuBLAS): {ms:.3f} ms {flops/ms/1e9:.1f} TFLOP/s")
