"""C1 context: cuBLAS at the C1 shape (1024^3 fp32), timed like bench.py (CUDA graph replays,
L2 flushed between steps): SGEMM (FFMA, the fp32-exact library path) and one TF32 pass, plus
torch's unfused LayerNorm -> SGEMM. Not product code: the comparison for the fp32 mode."""
import json
import torch

torch.backends.cuda.matmul.allow_tf32 = False
X = torch.randn(1024, 1024, device="cuda")
Y = torch.randn(1024, 1024, device="cuda")
flush = torch.empty(2 * 126 * 2**20 // 4, device="cuda")


def timed(fn, n=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    tot = 0.0
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n * 1e3  # us


res = {}
res["sgemm_fp32_us"] = timed(lambda: X @ Y.T)
torch.backends.cuda.matmul.allow_tf32 = True
res["tf32_one_pass_us"] = timed(lambda: X @ Y.T)
torch.backends.cuda.matmul.allow_tf32 = False
res["torch_layernorm_then_sgemm_us"] = timed(lambda: torch.nn.functional.layer_norm(X, (1024,), eps=0.0) @ Y.T)
for k in list(res):
    res[k.replace("_us", "_tflops")] = 2 * 1024**3 / (res[k] * 1e-6) / 1e12
print(json.dumps(res))
