"""Clock/power study at C2/C3/C4: each kernel run back to back for ~2 s with NVML sampling
(median SM clock and board power), next to its torch/cuBLAS/cuDNN counterpart. Answers whether
a kernel is held below the maximum SM clock by the power cap."""
import os, sys, threading, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import pynvml
from paper_2505_07829_b200 import ops

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1000,
                    pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.01)


def run(name, fn, flops, secs=2.0):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    t0 = time.time(); n = 0
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    stop = threading.Event(); smp = []
    th = threading.Thread(target=sample, args=(stop, smp)); th.start()
    e0.record()
    while time.time() - t0 < secs:
        fn(); n += 1
        if n % 8 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = e0.elapsed_time(e1) / n
    smp = smp[len(smp) // 4:]
    clk = sorted(c for c, _, _ in smp)[len(smp) // 2]; pw = sorted(p for _, p, _ in smp)[len(smp) // 2]
    reasons = 0
    for _, _, r in smp: reasons |= r
    print(f"{name}: {ms:.3f} ms/step {flops / ms / 1e9:.0f} TFLOP/s  median SM {clk} MHz  median power {pw:.0f} W  "
          f"reasons 0x{reasons:x}  {flops / ms / 1e9 / clk:.3f} TFLOP/s per MHz", flush=True)


which = sys.argv[1:] or ["attn", "ffn", "lnmm"]
if "attn" in which:
    B, H, S, D = 8, 32, 2048, 128
    Q = torch.randn(B * H, S, D, device="cuda").bfloat16(); K = torch.randn(B * H, S, D, device="cuda").bfloat16()
    Vt = torch.randn(B * H, D, S, device="cuda").bfloat16()
    fl = 4 * B * H * S * S * D
    run("K3 attention", lambda: ops.attention(Q, K, Vt), fl)
    q4, k4 = Q.view(B, H, S, D), K.view(B, H, S, D)
    v4 = Vt.transpose(1, 2).contiguous().view(B, H, S, D)
    run("torch SDPA (cuDNN)", lambda: torch.nn.functional.scaled_dot_product_attention(q4, k4, v4), fl)
if "ffn" in which:
    M, D, F = 8192, 4096, 14336
    X = torch.randn(M, D, device="cuda").bfloat16()
    Wt = (torch.randn(F, D, device="cuda") * D ** -0.5).bfloat16(); Vt = (torch.randn(F, D, device="cuda") * D ** -0.5).bfloat16()
    Ut = (torch.randn(D, F, device="cuda") * F ** -0.5).bfloat16()
    run("K1 fused C3", lambda: ops.rms_ffn_swiglu(X, Wt, Vt, Ut), 6 * M * D * F)
if "lnmm" in which:
    M, K, N = 65536, 4096, 4096
    X = torch.randn(M, K, device="cuda").bfloat16(); Yt = torch.randn(N, K, device="cuda").bfloat16()
    run("K2 C4", lambda: ops.layernorm_matmul(X, Yt), 2 * M * K * N)
    run("cuBLAS same shape", lambda: X @ Yt.T, 2 * M * K * N)
