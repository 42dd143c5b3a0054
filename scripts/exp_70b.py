"""C5 power study: fused K1 vs torch/cuBLAS unfused FFN at the Llama-3-70B shape (32768 tokens),
each run for ~2 s with NVML clock/power sampling."""
import sys, threading, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import pynvml
from paper_2505_07829_b200 import ops

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)

def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
        time.sleep(0.02)

def run(name, fn, flops, secs=2.0):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    t0 = time.time(); n = 0
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    stop = threading.Event(); smp = []
    th = threading.Thread(target=sample, args=(stop, smp)); th.start()
    e0.record()
    while time.time() - t0 < secs:
        fn(); n += 1
        if n % 4 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = e0.elapsed_time(e1) / n
    smp = smp[len(smp) // 4:]
    clk = sorted(c for c, _ in smp)[len(smp) // 2]; pw = sorted(p for _, p in smp)[len(smp) // 2]
    print(f"{name}: {ms:.2f} ms/step {flops / ms / 1e9:.0f} TFLOP/s  median SM {clk} MHz  median power {pw:.0f} W  ({n} steps)", flush=True)

M, D, F = 32768, 8192, 28672
X = torch.randn(M, D, device="cuda").bfloat16()
Wt = (torch.randn(F, D, device="cuda") * D ** -0.5).bfloat16(); Vt = (torch.randn(F, D, device="cuda") * D ** -0.5).bfloat16()
Ut = (torch.randn(D, F, device="cuda") * F ** -0.5).bfloat16()
fl = 6 * M * D * F
out = torch.empty(M, D, device="cuda", dtype=torch.bfloat16)
import os
which = os.environ.get("WHICH", "all")
if which == "fused":
    run(f"fused K1 (1SM={os.environ.get('BFGPU_FFN_1SM','0')}, group={os.environ.get('BFGPU_FFN_GROUP','default')})",
        lambda: ops.rms_ffn_swiglu(X, Wt, Vt, Ut, out=out), fl)
    sys.exit(0)
run("fused K1", lambda: ops.rms_ffn_swiglu(X, Wt, Vt, Ut, out=out), fl)
run("K1 two-phase", lambda: ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule="two_phase", out=out), fl)
def unfused():
    Xn = (X.float() * torch.rsqrt(X.float().square().mean(-1, keepdim=True))).bfloat16()
    return (torch.nn.functional.silu(Xn @ Wt.T) * (Xn @ Vt.T)) @ Ut.T
run("torch unfused", unfused, fl)
A = torch.randn(8192, 8192, device="cuda").bfloat16(); B = torch.randn(8192, 8192, device="cuda").bfloat16()
run("cuBLAS 8192^3", lambda: A @ B, 2 * 8192 ** 3)
