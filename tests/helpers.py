"""Shared test helpers: golden fixtures, bf16 rounding, and the parity metrics.

Tolerances (BASELINE.json north_star): bf16 inputs with fp32 accumulation must
match the float64 reference within max relative error 2e-2 (max|d| / max|ref|)
and max abs error 1e-2 on normalized outputs; fp32-in/fp32-out must match
within 1e-4 (max|d| / max|ref|). "Normalized" means divided by rms(ref), and
the abs bar is applied allclose-style, |d| <= 1e-2 + 2e-2 |ref| elementwise on
the normalized values: a bf16 OUTPUT alone carries up to
2^-9 |ref| of rounding, which at |ref| = 5 rms is already 1e-2. The reference's own
max_rel_error (interpreter.hpp:599-610, 1e-12 absolute floor) is meaningless
for bf16, so these metrics are stated here and used by every parity test.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

BF16_REL_TOL = 2e-2
BF16_NORM_ABS_TOL = 1e-2
F32_REL_TOL = 1e-4


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def bf16_round(a: np.ndarray) -> np.ndarray:
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def rel_err(out, ref) -> float:
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(out - ref)) / max(np.max(np.abs(ref)), 1e-300))


def norm_abs_err(out, ref) -> float:
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    rms = float(np.sqrt(np.mean(ref * ref)))
    return float(np.max(np.abs(out - ref)) / max(rms, 1e-300))


def norm_allclose_excess(out, ref, atol: float = BF16_NORM_ABS_TOL, rtol: float = BF16_REL_TOL) -> float:
    """max over elements of |d| - (atol + rtol |ref|) on rms-normalized values (<= 0 passes)."""
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    rms = max(float(np.sqrt(np.mean(ref * ref))), 1e-300)
    return float(np.max(np.abs(out - ref) / rms - (atol + rtol * np.abs(ref) / rms)))


def assert_bf16_close(out, ref, what: str = "", norm_tol: float = BF16_NORM_ABS_TOL) -> None:
    assert np.all(np.isfinite(out)), f"{what}: non-finite output"
    r, n = rel_err(out, ref), norm_abs_err(out, ref)
    assert r <= BF16_REL_TOL, f"{what}: max|d|/max|ref| = {r:.3e} > {BF16_REL_TOL}"
    ex = norm_allclose_excess(out, ref, atol=norm_tol)
    assert ex <= 0, f"{what}: normalized |d| exceeds {norm_tol} + 2e-2|ref| by {ex:.3e} (max|d|/rms = {n:.3e})"


def assert_f32_close(out, ref, what: str = "") -> None:
    assert np.all(np.isfinite(out)), f"{what}: non-finite output"
    r = rel_err(out, ref)
    assert r <= F32_REL_TOL, f"{what}: max|d|/max|ref| = {r:.3e} > {F32_REL_TOL}"


class DeviceErr:
    """The parity metrics above, accumulated on the GPU over chunks of a large output.

    Full-shape outputs (C2-C5) are compared element by element against a torch fp32
    reference computed on the device from the same bf16 inputs (TF32 off), without
    moving the output to the host: max|d|/max|ref| and the rms-normalized allclose
    excess max(|d| - rtol |ref|)/rms - atol."""

    def __init__(self, rtol: float = BF16_REL_TOL):
        self.rtol = rtol
        self.max_d = 0.0
        self.max_ref = 0.0
        self.max_dr = -float("inf")
        self.sq = 0.0
        self.n = 0
        self.nonfinite = 0

    def add(self, out, ref) -> None:
        import torch

        o = out.float()
        r = ref.float()
        d = (o - r).abs()
        self.nonfinite += int((~torch.isfinite(o)).sum().item())
        self.max_d = max(self.max_d, float(d.max().item()))
        self.max_ref = max(self.max_ref, float(r.abs().max().item()))
        self.max_dr = max(self.max_dr, float((d - self.rtol * r.abs()).max().item()))
        self.sq += float(r.double().pow(2).sum().item())
        self.n += r.numel()

    def summary(self) -> dict:
        rms = (self.sq / max(self.n, 1)) ** 0.5
        return {"rel": self.max_d / max(self.max_ref, 1e-300), "norm_abs": self.max_d / max(rms, 1e-300),
                "excess": self.max_dr / max(rms, 1e-300), "nonfinite": self.nonfinite, "elements": self.n}

    def check(self, what: str, norm_tol: float = BF16_NORM_ABS_TOL) -> dict:
        s = self.summary()
        print(f"{what}: {s}")
        assert s["nonfinite"] == 0, f"{what}: {s['nonfinite']} non-finite outputs"
        assert s["rel"] <= BF16_REL_TOL, f"{what}: max|d|/max|ref| = {s['rel']:.3e} > {BF16_REL_TOL}"
        assert s["excess"] - norm_tol <= 0, f"{what}: normalized |d| exceeds {norm_tol} + 2e-2|ref| ({s})"
        return s


def stratified_rows(M: int, unit: int, seed: int = 0) -> np.ndarray:
    """One row in every `unit`-row m-unit (the last, possibly ragged, unit included), at a
    random offset: every m-unit, scheduling group and raster block of a launch is hit."""
    rng = np.random.default_rng(seed)
    starts = np.arange(0, M, unit)
    return np.array([s + rng.integers(0, min(unit, M - s)) for s in starts], dtype=np.int64)
