"""Generate the golden fixtures in tests/golden/ from the reference itself.

Runs in the build container only: it needs oracle/_ref/libbfref.so, the
UNMODIFIED reference headers (/root/reference/proj/include) compiled in place
by oracle/Makefile. Inputs come from the reference's own random_inputs
(mt19937_64 N(0,1), interpreter.hpp:585) on the acceptance-suite seeds and
bindings (tests/acceptance.cpp:114-201, tests/test_engine.cpp:221-238), so the
fixtures pin the restated oracle and the GPU kernels to reference outputs.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import refexec as R  # noqa: E402

OUT = Path(__file__).resolve().parent


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bf16 (round-to-nearest-even), as float64."""
    f = a.astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def run_all_programs(which: int, inputs: dict, binding: dict, prefix: str, rec: dict) -> None:
    rec[f"{prefix}unfused"] = R.execute(which, R.UNFUSED, inputs, binding)
    for s in range(R.num_snapshots(which)):
        rec[f"{prefix}snap{s}"] = R.execute(which, s, inputs, binding)
    rec[f"{prefix}dense"] = R.dense(which, inputs)


def acceptance(which: int, name: str, binding: dict, seed0: int, trials: int = 3) -> None:
    rec: dict[str, np.ndarray] = {}
    for t in range(trials):
        inp = R.random_inputs(which, binding, seed0 + t)
        for k, v in inp.items():
            rec[f"t{t}_in_{k}"] = v
        run_all_programs(which, inp, binding, f"t{t}_", rec)
        if which == R.ATTENTION:
            for ch in (c for c in (1, 2, 4) if inp["K"].shape[0] % c == 0):
                rec[f"t{t}_safe{ch}"] = R.safe_attention(inp["Q"], inp["K"], inp["Vt"], ch)
    rec["binding"] = np.array(R.binding_str(binding).decode())
    rec["seeds"] = np.arange(seed0, seed0 + trials)
    np.savez_compressed(OUT / f"{name}.npz", **rec)


def gpu_sized(which: int, name: str, binding: dict, seed: int, row_scale: dict | None = None) -> None:
    """bf16-representable inputs at tensor-core tile sizes + reference outputs."""
    inp = R.random_inputs(which, binding, seed)
    for k in inp:
        s = (row_scale or {}).get(k, 1.0)
        inp[k] = bf16_round(inp[k] * s)
    rec = {f"in_{k}": v for k, v in inp.items()}
    rec["final"] = R.execute(which, R.FINAL, inp, binding)
    rec["dense"] = R.dense(which, inp)
    rec["binding"] = np.array(R.binding_str(binding).decode())
    rec["seed"] = np.array(seed)
    np.savez_compressed(OUT / f"{name}.npz", **rec)


def main() -> None:
    sq4 = lambda dims: {d: (2, 4) for d in dims}  # noqa: E731  bind_counts({...}, 4)
    acceptance(R.ATTENTION, "acceptance_attention", sq4("MNDL"), 1000)
    acceptance(R.LAYERNORM_MATMUL, "acceptance_layernorm_matmul", sq4("MNK"), 2000)
    acceptance(R.RMS_FFN_SWIGLU, "acceptance_rms_ffn_swiglu", sq4("MKND"), 3000)
    asym = {"M": (3, 2), "N": (2, 3), "D": (1, 4), "L": (2, 2), "K": (4, 2)}
    acceptance(R.ATTENTION, "asymmetric_attention", asym, 5, trials=2)
    acceptance(R.RMS_FFN_SWIGLU, "asymmetric_rms_ffn_swiglu", asym, 6, trials=2)
    # tensor-core sized cases (multiples of the 128-row tiles plus partial blocks)
    gpu_sized(R.RMS_FFN_SWIGLU, "gpu_rms_ffn_swiglu", {"M": (3, 64), "D": (2, 128), "K": (3, 128), "N": (2, 128)}, 31,
              row_scale={"Wt": 1 / 16, "Vt": 1 / 16, "Ut": 1 / 16})
    gpu_sized(R.LAYERNORM_MATMUL, "gpu_layernorm_matmul", {"M": (3, 64), "K": (2, 128), "N": (3, 128)}, 32)
    gpu_sized(R.ATTENTION, "gpu_attention", {"M": (2, 128), "N": (3, 128), "D": (1, 128), "L": (1, 128)}, 33)
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
