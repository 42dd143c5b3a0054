"""C1 (LN->MM fp32, 1024^3) per-launch durations, warm: run under
`ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum`.
Also prints the CUDA-event time per call (graph replay, no L2 flush) when run plain."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_07829_b200 import ops

g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(1024, 1024, device="cuda", generator=g)
Yt = torch.randn(1024, 1024, device="cuda", generator=g)
O = ops.layernorm_matmul(X, Yt)
torch.cuda.synchronize()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        ops.layernorm_matmul(X, Yt)
    s.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(20):
            ops.layernorm_matmul(X, Yt)
    gr.replay()
    s.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(s)
    for _ in range(10):
        gr.replay()
    b.record(s)
    s.synchronize()
print(f"C1 warm graph replay: {a.elapsed_time(b) / 200 * 1e3:.1f} us per call")
