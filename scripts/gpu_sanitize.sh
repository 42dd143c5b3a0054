#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small calls of every plan.
mkdir -p gpurun_out
cat > /tmp/san.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2505_07829_b200 import ops
g = torch.Generator(device="cuda").manual_seed(0)
r = lambda *s: torch.randn(*s, device="cuda", generator=g).bfloat16()
X, Wt, Vt, Ut = r(520, 256), r(392, 256) * 0.06, r(392, 256) * 0.06, r(264, 392) * 0.05
for s in ("fused", "two_phase"):
    ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule=s)
Xl, Yt = r(600, 264) + 1, r(392, 264)
for s in ("fused", "staged"):
    ops.layernorm_matmul(Xl, Yt, schedule=s)
ops.layernorm_matmul(Xl.float(), Yt.float())
Q, K, Vv = r(3, 300, 128), r(3, 456, 128), r(3, 128, 456)
for s in ("fused", "staged"):
    ops.attention(Q, K, Vv, schedule=s)
ops.attention(Q.float(), K.float(), Vv.float())
ops.rms_ffn_swiglu(X.float(), Wt.float(), Vt.float(), Ut.float())
import os
os.environ["BFGPU_F32_BN"] = "256"  # the 128x256-tile 3xTF32 GEMMs at a small shape
ops.layernorm_matmul(Xl.float(), Yt.float())
ops.rms_ffn_swiglu(X.float(), Wt.float(), Vt.float(), Ut.float())
ops.attention(Q.float()[:, :, :64].contiguous(), K.float()[:, :, :64].contiguous(), Vv.float()[:, :64].contiguous())
torch.cuda.synchronize()
print("san ok")
PY
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san.py > gpurun_out/san_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -6 gpurun_out/san_$tool.log
done
