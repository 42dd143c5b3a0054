"""fp32 attention (3xTF32 tensor-core plan) against float64 on a few shapes; prints the plan kernel."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_07829_b200 import ops

CASES = [(1, 128, 64, 128, 128), (2, 200, 136, 64, 128), (3, 77, 1000, 128, 64), (2, 300, 2048, 64, 64),
         (4, 1024, 4096, 128, 128), (1, 128, 128, 128, 128), (1, 128, 256, 128, 128), (2, 256, 2048, 128, 128)]
sel = [int(a) for a in sys.argv[1:]] or range(len(CASES))
for BH, Sq, Skv, D, Dv in [CASES[i] for i in sel]:
    g = torch.Generator(device="cuda").manual_seed(BH * 7 + Sq)
    Q = torch.randn(BH, Sq, D, device="cuda", generator=g) * 2
    K = torch.randn(BH, Skv, D, device="cuda", generator=g)
    Vt = torch.randn(BH, Dv, Skv, device="cuda", generator=g)
    kern = ops.plan("attention", (BH, Sq, Skv, D, Dv), dtype=torch.float32)["kernel"]
    O = ops.attention(Q, K, Vt)
    torch.cuda.synchronize()
    ref = torch.softmax(Q.double() @ K.double().transpose(1, 2) / D ** 0.5, -1) @ Vt.double().transpose(1, 2)
    err = float((O.double() - ref).abs().max() / ref.abs().max())
    print(f"{kern} BH={BH} Sq={Sq} Skv={Skv} D={D} Dv={Dv}: max|d|/max|ref| = {err:.2e}", flush=True)
