"""Scratch: device timing of K1/K2/K3 at the BASELINE configs + torch/cuBLAS baselines."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_07829_b200 import ops

def timeit(fn, n=10, w=3):
    for _ in range(w): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

which = sys.argv[1:] or ["ffn", "lnmm", "attn"]
if "ffn" in which:
    M, D, F = 8192, 4096, 14336
    X = torch.randn(M, D, device="cuda").bfloat16()
    Wt = (torch.randn(F, D, device="cuda") * 0.02).bfloat16(); Vt = (torch.randn(F, D, device="cuda") * 0.02).bfloat16()
    Ut = (torch.randn(D, F, device="cuda") * 0.02).bfloat16()
    fl = 6 * M * D * F
    for s in ("two_phase", "fused"):
        ms = timeit(lambda: ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule=s))
        print(f"K1 {s}: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)
if "lnmm" in which:
    M, K, N = 65536, 4096, 4096
    X = torch.randn(M, K, device="cuda").bfloat16(); Yt = torch.randn(N, K, device="cuda").bfloat16()
    fl = 2 * M * K * N
    ms = timeit(lambda: ops.layernorm_matmul(X, Yt))
    print(f"K2: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)
    ms = timeit(lambda: torch.nn.functional.layer_norm(X, (K,)) @ Yt.T)
    print(f"K2 torch unfused: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)
    ms = timeit(lambda: X @ Yt.T)
    print(f"cuBLAS plain GEMM same shape: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)
if "attn" in which:
    B, H, S, D = 8, 32, 2048, 128
    Q = torch.randn(B, H, S, D, device="cuda").bfloat16(); Kk = torch.randn(B, H, S, D, device="cuda").bfloat16()
    Vt = torch.randn(B, H, D, S, device="cuda").bfloat16()
    fl = 4 * B * H * S * S * D
    ms = timeit(lambda: ops.attention(Q, Kk, Vt))
    print(f"K3: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)
    V = Vt.transpose(-1, -2).contiguous()
    ms = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(Q, Kk, V))
    print(f"torch SDPA: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)
