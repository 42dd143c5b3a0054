"""Minimal launcher for ncu captures: runs one workload's kernel `n` times at the BASELINE shape."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import WORKLOADS, make_inputs, step_fn

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "ffn_8b"]
sched = sys.argv[2] if len(sys.argv) > 2 else "fused"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 3
inp = make_inputs(wl, 0, 1, torch.device("cuda", 0))
if wl["kind"] == "attn":
    out = torch.empty_like(inp["Q"])
else:
    out = torch.empty(inp["rows"], wl["N"], dtype=inp["X"].dtype, device="cuda")
fn = step_fn(wl, inp, sched, out)
for _ in range(n):
    fn()
torch.cuda.synchronize()
print("done", wl["name"], sched)
