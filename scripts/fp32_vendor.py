"""fp32 modes against the vendor fp32 paths at the same shapes (CUDA events, 3 warm-up + 5 timed):
K3 C2 shape vs torch SDPA on fp32 inputs (TF32 off), K1 C3 shape vs torch fp32 (RMSNorm, two
SGEMMs, SiLU*mul, SGEMM), K2 C4 shape vs torch LayerNorm + SGEMM. Prints JSON lines."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import torch.nn.functional as Fn
from paper_2505_07829_b200 import ops

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False


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
Q, K, V = r(8, 32, 2048, 128), r(8, 32, 2048, 128), r(8, 32, 2048, 128)
Vt = V.transpose(-1, -2).contiguous()
fl = 4 * 256 * 2048 * 2048 * 128
ours = t(lambda: ops.attention(Q, K, Vt))
sdpa = t(lambda: Fn.scaled_dot_product_attention(Q, K, V))
print(json.dumps({"op": "K3 fp32 C2", "ours_ms": round(ours, 3), "ours_tflops": round(fl / ours / 1e9, 1),
                  "torch_sdpa_fp32_ms": round(sdpa, 3), "torch_sdpa_tflops": round(fl / sdpa / 1e9, 1)}))
del Q, K, V, Vt
M, D, F = 8192, 4096, 14336
X, Wt, Wv, Ut = r(M, D), r(F, D) * D ** -0.5, r(F, D) * D ** -0.5, r(D, F) * F ** -0.5


def torch_ffn():
    Xn = X * torch.rsqrt(X.pow(2).mean(-1, keepdim=True))
    return (Fn.silu(Xn @ Wt.T) * (Xn @ Wv.T)) @ Ut.T


fl = 6 * M * D * F
ours = t(lambda: ops.rms_ffn_swiglu(X, Wt, Wv, Ut))
ref = t(torch_ffn)
print(json.dumps({"op": "K1 fp32 C3", "ours_ms": round(ours, 3), "ours_tflops": round(fl / ours / 1e9, 1),
                  "torch_fp32_ms": round(ref, 3), "torch_tflops": round(fl / ref / 1e9, 1)}))
del X, Wt, Wv, Ut
X, Yt = r(65536, 4096), r(4096, 4096)
fl = 2 * 65536 * 4096 * 4096
ours = t(lambda: ops.layernorm_matmul(X, Yt))
ref = t(lambda: Fn.layer_norm(X, (4096,)) @ Yt.T)
print(json.dumps({"op": "K2 fp32 C4", "ours_ms": round(ours, 3), "ours_tflops": round(fl / ours / 1e9, 1),
                  "torch_fp32_ms": round(ref, 3), "torch_tflops": round(fl / ref / 1e9, 1)}))
