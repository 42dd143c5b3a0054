"""K1 Flash-RMSNorm+FFN-SwiGLU on the B200 vs the reference (GPU parity tests).

Oracle: the reference executor's output on the final fused snapshot
(tests/golden/, made by tests/golden/make_golden.py from the unmodified
reference) and the C restatement (oracle/bf_oracle.c) at other shapes.
Mirrors tests/acceptance.cpp:175-201 (criterion 4) and
tests/test_engine.cpp:221-238 (asymmetric bindings) of the reference.
"""
import numpy as np
import pytest

from helpers import assert_bf16_close, assert_f32_close, bf16_round, golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_ops():
    import torch

    from paper_2505_07829_b200 import ops

    return torch, ops


def _dev(torch, a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def _run(torch, ops, X, Wt, Vt, Ut, dtype, **kw):
    args = [_dev(torch, a, dtype) for a in (X, Wt, Vt, Ut)]
    out = ops.rms_ffn_swiglu(*args, **kw)
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


@pytest.mark.parametrize("schedule", ["fused", "two_phase"])
def test_golden_final_snapshot_bf16(torch_ops, schedule):
    torch, ops = torch_ops
    g = golden("gpu_rms_ffn_swiglu")
    out = _run(torch, ops, g["in_X"], g["in_Wt"], g["in_Vt"], g["in_Ut"], torch.bfloat16, schedule=schedule)
    assert_bf16_close(out, g["final"], f"K1 {schedule} vs reference execute(final snapshot)")
    assert_bf16_close(out, g["dense"], f"K1 {schedule} vs ref::rms_ffn_swiglu")


@pytest.mark.parametrize("fixture", ["acceptance_rms_ffn_swiglu", "asymmetric_rms_ffn_swiglu"])
def test_golden_fp32_mode(torch_ops, fixture):
    """fp32-in/fp32-out must match the float64 reference within 1e-4 (any shape)."""
    torch, ops = torch_ops
    g = golden(fixture)
    t = 0
    while f"t{t}_in_X" in g:
        out = _run(torch, ops, g[f"t{t}_in_X"], g[f"t{t}_in_Wt"], g[f"t{t}_in_Vt"], g[f"t{t}_in_Ut"], torch.float32)
        n_snap = sum(1 for k in g if k.startswith(f"t{t}_snap"))
        assert_f32_close(out, g[f"t{t}_snap{n_snap - 1}"], f"{fixture} trial {t} vs final snapshot")
        assert_f32_close(out, g[f"t{t}_unfused"], f"{fixture} trial {t} vs unfused program")
        t += 1
    assert t > 0


@pytest.mark.parametrize(
    "M,D,F,N",
    [(1, 64, 128, 64), (128, 64, 128, 256), (300, 200, 136, 264), (513, 512, 1032, 520), (2048, 256, 512, 256)],
)
def test_ragged_shapes_vs_oracle(torch_ops, M, D, F, N):
    torch, ops = torch_ops
    from oracle import cpu

    rng = np.random.default_rng(M * 7 + D)
    X = bf16_round(rng.standard_normal((M, D)))
    Wt = bf16_round(rng.standard_normal((F, D)) / np.sqrt(D))
    Vt = bf16_round(rng.standard_normal((F, D)) / np.sqrt(D))
    Ut = bf16_round(rng.standard_normal((N, F)) / np.sqrt(F))
    ref = cpu.rms_ffn_swiglu(X, Wt, Vt, Ut)
    for sched in ("fused", "two_phase"):
        out = _run(torch, ops, X, Wt, Vt, Ut, torch.bfloat16, schedule=sched)
        assert_bf16_close(out, ref, f"K1 {sched} {M}x{D}x{F}x{N}")
    out32 = _run(torch, ops, X, Wt, Vt, Ut, torch.float32)
    assert_f32_close(out32, ref, f"K1 fp32 {M}x{D}x{F}x{N}")


def test_eps(torch_ops):
    torch, ops = torch_ops
    from oracle import cpu

    rng = np.random.default_rng(5)
    M, D, F, N = 256, 128, 256, 128
    X = bf16_round(rng.standard_normal((M, D)) * 1e-2)
    Wt, Vt = (bf16_round(rng.standard_normal((F, D)) / 8) for _ in range(2))
    Ut = bf16_round(rng.standard_normal((N, F)) / 16)
    ref = cpu.rms_ffn_swiglu(X, Wt, Vt, Ut, eps=1e-3)
    out = _run(torch, ops, X, Wt, Vt, Ut, torch.bfloat16, eps=1e-3)
    assert_bf16_close(out, ref, "K1 eps=1e-3")


def test_fused_equals_two_phase_bitwise(torch_ops):
    """Both schedules run identical tile arithmetic; only the H hand-off differs."""
    torch, ops = torch_ops
    g = torch.Generator(device="cuda").manual_seed(1)
    M, D, F = 4096, 1024, 2816
    X = torch.randn(M, D, device="cuda", generator=g).bfloat16()
    Wt, Vt = (torch.randn(F, D, device="cuda", generator=g).mul(0.03).bfloat16() for _ in range(2))
    Ut = torch.randn(D, F, device="cuda", generator=g).mul(0.02).bfloat16()
    a = ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule="fused")
    b = ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule="two_phase")
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_llama3_8b_shape_properties(torch_ops):
    """C3 (d=4096, ffn=14336, 8192 tokens): sampled rows vs the oracle, and the
    RMSNorm scale invariance O(2X) == O(X) (exact in binary floating point)."""
    torch, ops = torch_ops
    from oracle import cpu

    g = torch.Generator(device="cuda").manual_seed(2)
    M, D, F = 8192, 4096, 14336
    X = torch.randn(M, D, device="cuda", generator=g).bfloat16()
    Wt, Vt = (torch.randn(F, D, device="cuda", generator=g).mul(D ** -0.5).bfloat16() for _ in range(2))
    Ut = torch.randn(D, F, device="cuda", generator=g).mul(F ** -0.5).bfloat16()
    O = ops.rms_ffn_swiglu(X, Wt, Vt, Ut)
    O2 = ops.rms_ffn_swiglu(X * 2, Wt, Vt, Ut)
    torch.cuda.synchronize()
    assert torch.equal(O, O2)
    rows = torch.tensor([0, 1, 127, 128, 4095, 5000, 8190, 8191], device="cuda")
    ref = cpu.rms_ffn_swiglu(X[rows].double().cpu().numpy(), Wt.double().cpu().numpy(), Vt.double().cpu().numpy(),
                             Ut.double().cpu().numpy())
    assert_bf16_close(O[rows].double().cpu().numpy(), ref, "K1 8B sampled rows")


def test_errors_are_loud(torch_ops):
    torch, ops = torch_ops
    from paper_2505_07829_b200 import BfError

    X = torch.zeros(4, 12, device="cuda", dtype=torch.bfloat16)  # D not a multiple of 8
    W = torch.zeros(16, 12, device="cuda", dtype=torch.bfloat16)
    U = torch.zeros(12, 16, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(BfError):
        ops.rms_ffn_swiglu(X, W, W, U)
