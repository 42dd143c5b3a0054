"""Seeded random shape sweep of every plan, both dtypes and both schedules.

The parity tests elsewhere pin the BASELINE shapes and hand-picked ragged ones; this sweep
draws sizes that are NOT multiples of the tiles (rows, heads, query and key lengths, every
contraction and output width a random multiple of 8, the C-ABI's only alignment rule) and
checks each call against the fp32 torch reference on the same inputs (tests/torch_ref.py), in
the north star's tolerances (tests/helpers.py): bf16 max|d|/max|ref| <= 2e-2 plus the
rms-normalized allclose, fp32 <= 1e-4. The sizes mirror the reference's interpreter tests,
which bind every dimension independently (tests/test_engine.cpp:221-238).
"""
import numpy as np
import pytest

import torch_ref
from helpers import F32_REL_TOL, DeviceErr

pytestmark = pytest.mark.gpu

CASES = 24


@pytest.fixture(scope="module")
def torch_ops():
    import torch

    from paper_2505_07829_b200 import ops

    return torch, ops


def _rand(torch, shape, scale, dtype, g):
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(dtype)


def _check(torch, outs, refs, dtype, what):
    if dtype == torch.bfloat16:
        e = DeviceErr()
        for o, r in zip(outs, refs):
            e.add(o, r)
        e.check(what)
    else:
        md = max(float((o.float() - r).abs().max()) for o, r in zip(outs, refs))
        mr = max(float(r.abs().max()) for r in refs)
        assert md / mr <= F32_REL_TOL, f"{what}: max|d|/max|ref| = {md / mr:.3e}"


def _m8(rng, lo, hi):
    return int(rng.integers(lo // 8, hi // 8 + 1)) * 8


@pytest.mark.parametrize("case", range(CASES))
def test_ffn_random_shapes(torch_ops, case):
    torch, ops = torch_ops
    rng = np.random.default_rng(100 + case)
    dtype = torch.bfloat16 if case % 3 else torch.float32
    M = int(rng.integers(1, 1300))
    D, F, N = _m8(rng, 8, 1024), _m8(rng, 8, 1600), _m8(rng, 8, 1024)
    g = torch.Generator(device="cuda").manual_seed(case)
    X = _rand(torch, (M, D), 1.0, dtype, g)
    Wt, Vt = _rand(torch, (F, D), D ** -0.5, dtype, g), _rand(torch, (F, D), D ** -0.5, dtype, g)
    Ut = _rand(torch, (N, F), F ** -0.5, dtype, g)
    refs = [r for _, r in torch_ref.rms_ffn_swiglu_chunks(X, Wt, Vt, Ut, chunk=1 << 20)]
    scheds = ("fused", "two_phase") if dtype == torch.bfloat16 else ("fused",)
    for s in scheds:
        O = ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule=s)
        torch.cuda.synchronize()
        _check(torch, [O], refs, dtype, f"K1 {s} {dtype} M={M} D={D} F={F} N={N}")


@pytest.mark.parametrize("case", range(CASES))
def test_lnmm_random_shapes(torch_ops, case):
    torch, ops = torch_ops
    rng = np.random.default_rng(200 + case)
    dtype = torch.bfloat16 if case % 3 else torch.float32
    M = int(rng.integers(1, 2500))
    K, N = _m8(rng, 8, 1600), _m8(rng, 8, 1400)
    g = torch.Generator(device="cuda").manual_seed(case)
    X = _rand(torch, (M, K), 1.0, dtype, g) + float(rng.uniform(-3, 3))  # off-centre rows
    Yt = _rand(torch, (N, K), 1.0, dtype, g)
    refs = [r for _, r in torch_ref.layernorm_matmul_chunks(X, Yt, chunk=1 << 20)]
    scheds = ("fused", "staged") if dtype == torch.bfloat16 else ("fused",)
    for s in scheds:
        O = ops.layernorm_matmul(X, Yt, schedule=s)
        torch.cuda.synchronize()
        _check(torch, [O], refs, dtype, f"K2 {s} {dtype} M={M} K={K} N={N}")


@pytest.mark.parametrize("case", range(CASES))
def test_attention_random_shapes(torch_ops, case):
    torch, ops = torch_ops
    rng = np.random.default_rng(300 + case)
    dtype = torch.bfloat16 if case % 3 else torch.float32
    BH = int(rng.integers(1, 7))
    Sq = int(rng.integers(1, 700))
    Skv = _m8(rng, 8, 900)
    D, Dv = (int(rng.choice([64, 128])), int(rng.choice([64, 128]))) if dtype == torch.bfloat16 else (
        _m8(rng, 8, 128), _m8(rng, 8, 128))
    g = torch.Generator(device="cuda").manual_seed(case)
    Q = _rand(torch, (BH, Sq, D), 1.0, dtype, g)
    K = _rand(torch, (BH, Skv, D), 1.0, dtype, g)
    Vt = _rand(torch, (BH, Dv, Skv), 1.0, dtype, g)
    refs = [r for _, r in torch_ref.attention_chunks(Q, K, Vt, heads=1 << 20)]
    scheds = ("fused", "staged") if dtype == torch.bfloat16 else ("fused",)
    for s in scheds:
        O = ops.attention(Q, K, Vt, schedule=s)
        torch.cuda.synchronize()
        _check(torch, [O], refs, dtype, f"K3 {s} {dtype} BH={BH} Sq={Sq} Skv={Skv} D={D} Dv={Dv}")
