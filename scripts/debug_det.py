import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_07829_b200 import ops
torch.manual_seed(0)
def tiles_differ(a, b, bm=128, bn=256):
    d = (a != b)
    M, N = d.shape
    t = d[: M // bm * bm, : N // bn * bn].reshape(M // bm, bm, N // bn, bn).sum((1, 3))
    return t
for (M, K, N) in [(128 * 148, 4096, 256), (128 * 148, 4096, 512), (8192, 4096, 4096), (8192, 256, 4096)]:
    X = torch.randn(M, K, device="cuda").bfloat16(); Yt = torch.randn(N, K, device="cuda").bfloat16()
    outs = [ops.layernorm_matmul(X, Yt).clone() for _ in range(3)]
    torch.cuda.synchronize()
    ref = (torch.nn.functional.layer_norm(X.float(), (K,)) @ Yt.float().T)
    for i in (1, 2):
        t = tiles_differ(outs[0], outs[i])
        nz = t.nonzero()
        print(f"K2 {M}x{K}x{N} run0 vs run{i}: {int((outs[0]!=outs[i]).sum())} elems differ in {len(nz)} tiles; first tiles {nz[:6].tolist()}", flush=True)
    print("   err vs torch fp32:", ((outs[0].float() - ref).abs().max() / ref.abs().max()).item())
# gemm-only probe: Yt with constant rows -> stats irrelevant? use X with zero-mean unit rows
