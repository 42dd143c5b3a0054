"""The reference's traffic model (traffic_bytes, metrics.hpp:154-191) at every bench workload
and at the bindings of scripts/snapshot_traffic.py, written to tests/golden/traffic_model.json.

Runs in the build container only (oracle/_ref/libbfref.so = the reference headers compiled in
place). bench.py and the snapshot-traffic script read the JSON; neither touches oracle/ at run
time. The model is exact integer arithmetic over the program structure, so these numbers are
the reference's own, not a restatement.

    python tests/golden/make_traffic_model.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import refexec as R  # noqa: E402

OUT = Path(__file__).resolve().parent / "traffic_model.json"

# bench workloads: M counted in 128-row blocks, every contraction dimension one block
# (counts = 1), the binding the fused kernels' tiles do not depend on
BENCH = {
    "ffn_8b": ("rms-swiglu", {"N": (1, 4096), "K": (1, 14336), "D": (1, 4096)}),
    "ffn_70b": ("rms-swiglu", {"N": (1, 8192), "K": (1, 28672), "D": (1, 8192)}),
    "lnmm": ("layernorm-matmul", {"K": (1, 4096), "N": (1, 4096)}),
    "lnmm_c1": ("layernorm-matmul", {"K": (1, 1024), "N": (1, 1024)}),
    "attn": ("attention", {"N": (1, 2048), "D": (1, 128), "L": (1, 128)}),  # per head, M = 16 x 128
}
WHICH = {"rms-swiglu": R.RMS_FFN_SWIGLU, "layernorm-matmul": R.LAYERNORM_MATMUL, "attention": R.ATTENTION}

# scripts/snapshot_traffic.py: one GPU run per program file. "generic" = every program file
# (lowered + each snapshot) on the float64 block-program compiler route (element_bytes 8);
# "kernels" = the snapshots on their bf16 tensor-core plans (element_bytes 2), larger.
RUNS = {
    "rms-swiglu": {"generic": "M=4,N=1,K=1,D=1 --len M=128,N=512,K=1024,D=512",
                   "kernels": "M=32,N=1,K=1,D=1 --len M=128,N=4096,K=14336,D=4096"},
    "layernorm-matmul": {"generic": "M=4,K=1,N=1 --len M=128,K=512,N=512",
                         "kernels": "M=128,K=1,N=1 --len M=128,K=4096,N=4096"},
    "attention": {"generic": "M=4,N=1,D=1,L=1 --len M=128,N=512,D=128,L=128",
                  "kernels": "M=16,N=1,D=1,L=1 --len M=128,N=2048,D=128,L=128"},
}


def parse_run(spec: str) -> dict:
    dims, lens = spec.split(" --len ")
    counts = {k: int(v) for k, v in (p.split("=") for p in dims.split(","))}
    ln = {k: int(v) for k, v in (p.split("=") for p in lens.split(","))}
    return {k: (counts[k], ln[k]) for k in counts}


def programs(which: int) -> dict[str, int]:
    out = {"lowered": R.UNFUSED}
    for s in range(R.num_snapshots(which)):
        out[f"snapshot_{s + 1}"] = s
    return out


def main() -> None:
    assert R.available(), "build oracle/_ref first (make -C oracle)"
    res = {"source": "traffic_bytes (metrics.hpp:154-191) of the reference compiled in place (oracle/_ref)",
           "bench_affine_in_m": {}, "runs": {}}
    for w, (ex, b) in BENCH.items():
        which = WHICH[ex]
        eb = 4 if w == "lnmm_c1" else 2
        ent = {"example": ex, "element_bytes": eb, "binding_besides_M": {k: list(v) for k, v in b.items()}}
        for name, snap in programs(which).items():
            # affine in the M count (per-m traffic + what the program reads once, e.g. broadcast
            # operands of unfused maps): model(m) = base + m * per_m; checked at a third point
            one = R.traffic_bytes(which, snap, {**b, "M": (1, 128)}, eb)
            two = R.traffic_bytes(which, snap, {**b, "M": (2, 128)}, eb)
            five = R.traffic_bytes(which, snap, {**b, "M": (5, 128)}, eb)
            assert five == one + 4 * (two - one), f"{w} {name}: model not affine in the M count"
            ent[name] = {"per_m_block": two - one, "base": 2 * one - two}
        res["bench_affine_in_m"][w] = ent
    for ex, specs in RUNS.items():
        which = WHICH[ex]
        ent = {"spec": specs, "model_bytes": {}}
        for route, eb in (("generic", 8), ("kernels", 2)):
            b = parse_run(specs[route])
            ent["model_bytes"][route] = {name: R.traffic_bytes(which, snap, b, eb)
                                         for name, snap in programs(which).items()}
        ent["internal_buffered_edges"] = {name: R.program_stats(which, snap)["internal_buffered"]
                                          for name, snap in programs(which).items()}
        ent["kernels"] = {name: R.program_stats(which, snap)["kernels"] for name, snap in programs(which).items()}
        res["runs"][ex] = ent
    OUT.write_text(json.dumps(res, indent=1, sort_keys=True) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
