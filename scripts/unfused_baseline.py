"""Measured "HBM bytes vs unfused": the operator-by-operator sequence of each block program
(one library kernel per top-level operator of the reference's unfused lower() program,
bf/lowering.hpp:498-550), timed with CUDA events and, under ncu, its DRAM bytes summed over
every kernel of one step.

    python scripts/unfused_baseline.py time                 # -> JSON lines with ms and TFLOP/s
    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --csv --log-file gpurun_out/unfused_<w>.csv python scripts/unfused_baseline.py ncu <w>
    python scripts/unfused_baseline.py summarize gpurun_out/unfused_*.csv   # -> profiles/unfused_baseline.json

The unfused sequences use torch/cuBLAS kernels: this is the baseline the fused kernels are
compared against, not product code.
"""
from __future__ import annotations

import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

WL = ["ffn_8b", "lnmm", "attn"]


def sequences(w, inp):
    import torch

    if w.startswith("ffn"):
        X, Wt, Vt, Ut = inp["X"], inp["Wt"], inp["Vt"], inp["Ut"]

        def run():
            r = torch.rsqrt(X.float().square().mean(-1, keepdim=True))  # rmsnorm statistics (eps = 0)
            Xn = (X.float() * r).bfloat16()                                 # rmsnorm -> Xn in HBM
            G = Xn @ Wt.T                                                   # gate GEMM
            U = Xn @ Vt.T                                                   # up GEMM
            H = torch.nn.functional.silu(G) * U                             # swish * up
            return H @ Ut.T                                                 # down GEMM
        return run
    if w == "lnmm":
        X, Yt = inp["X"], inp["Yt"]

        def run():
            Xn = torch.nn.functional.layer_norm(X, (X.shape[-1],), eps=0.0)  # no gamma/beta, eps = 0
            return Xn @ Yt.T
        return run
    Q, K, Vt = inp["Q"], inp["K"], inp["Vt"]

    def run():
        S = (Q @ K.transpose(-1, -2)) * (Q.shape[-1] ** -0.5)  # S materialized
        P = torch.softmax(S.float(), -1).bfloat16()              # P materialized
        return P @ Vt.transpose(-1, -2)
    return run


def setup(w):
    import torch
    from bench import WORKLOADS, make_inputs

    wl = WORKLOADS[w]
    inp = make_inputs(wl, 0, 1, torch.device("cuda", 0))
    if w == "attn":  # keep the S x S intermediates within memory: 1/8 of the heads, scaled back up
        inp = {k: (v[:32] if hasattr(v, "dim") and v.dim() == 3 else v) for k, v in inp.items()}
        inp["flops"] = inp["flops"] / 8
    return wl, inp


def time_all():
    import torch

    for w in WL:
        wl, inp = setup(w)
        fn = sequences(w, inp)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        n = 10
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(json.dumps({"workload": w, "ms": ms, "tflops": inp["flops"] / ms / 1e9,
                          "sample": "32 of 256 heads; TFLOP/s on that sample" if w == "attn" else "full"}))


def ncu_one(w):
    import torch

    _, inp = setup(w)
    fn = sequences(w, inp)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    fn()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


def summarize(paths):
    out_p = ROOT / "profiles" / "unfused_baseline.json"
    summ = json.loads(out_p.read_text()) if out_p.exists() else {}
    for path in paths:
        w = Path(path).stem.replace("unfused_", "")
        lines = Path(path).read_text().splitlines()
        start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
        rows = list(csv.reader(lines[start:]))
        h = rows[0]
        ik, im, iu, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
        tot = {"dram": 0.0, "time_s": 0.0}
        kernels = set()
        for r in rows[1:]:
            v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
            kernels.add(r[0])
            if r[im].startswith("dram__bytes"):
                tot["dram"] += v
            elif r[im] == "gpu__time_duration.sum":
                tot["time_s"] += v
        factor = 8 if w == "attn" else 1  # attention sample = 1/8 of the heads
        summ[w] = {"dram_bytes_per_step": tot["dram"] * factor, "kernels": len(kernels),
                   "serialized_kernel_time_s": tot["time_s"] * factor,
                   "source": f"ncu dram__bytes_read+write over every kernel of one unfused step ({Path(path).name})"
                   + ("; measured on 1/8 of the heads, scaled x8" if w == "attn" else "")}
    out_p.write_text(json.dumps(summ, indent=1, sort_keys=True) + "\n")
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "time":
        time_all()
    elif cmd == "ncu":
        ncu_one(sys.argv[2])
    else:
        summarize(sys.argv[2:])
