"""K2 Flash-LayerNorm+MatMul on the B200 vs the reference (GPU parity tests).

Mirrors tests/acceptance.cpp:135-173 (criterion 3). The fused program computes
(X Yt^T - mu colsum(Yt)) * rstd on raw X; sigma = 0 rows are undefined (NaN)
in the fused reference walk, so test data is Gaussian like the reference's.
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


def _run(torch, ops, X, Yt, dtype, **kw):
    x = torch.from_numpy(np.ascontiguousarray(X)).to("cuda", dtype)
    y = torch.from_numpy(np.ascontiguousarray(Yt)).to("cuda", dtype)
    out = ops.layernorm_matmul(x, y, **kw)
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


def test_golden_final_snapshot_bf16(torch_ops):
    torch, ops = torch_ops
    g = golden("gpu_layernorm_matmul")
    out = _run(torch, ops, g["in_X"], g["in_Yt"], torch.bfloat16)
    assert_bf16_close(out, g["final"], "K2 vs reference execute(final snapshot)")
    assert_bf16_close(out, g["dense"], "K2 vs ref::layernorm_matmul")


def test_golden_fp32_mode(torch_ops):
    torch, ops = torch_ops
    g = golden("acceptance_layernorm_matmul")
    for t in range(3):
        out = _run(torch, ops, g[f"t{t}_in_X"], g[f"t{t}_in_Yt"], torch.float32)
        assert_f32_close(out, g[f"t{t}_snap1"], f"trial {t} vs final snapshot")
        assert_f32_close(out, g[f"t{t}_dense"], f"trial {t} vs ref::layernorm_matmul")


def test_c1_fp32_1024(torch_ops):
    """C1: M=K=N=1024 fp32, the reference's CPU-runnable config; 1e-4 vs the float64 oracle."""
    torch, ops = torch_ops
    from oracle import cpu

    rng = np.random.default_rng(2000)
    X = rng.standard_normal((1024, 1024)).astype(np.float32).astype(np.float64)
    Yt = rng.standard_normal((1024, 1024)).astype(np.float32).astype(np.float64)
    out = _run(torch, ops, X, Yt, torch.float32)
    assert_f32_close(out, cpu.layernorm_matmul(X, Yt), "C1 fp32")


@pytest.mark.parametrize("M,K,N", [(1, 64, 256), (200, 136, 264), (384, 512, 512), (1000, 1024, 776)])
def test_ragged_shapes_vs_oracle(torch_ops, M, K, N):
    torch, ops = torch_ops
    from oracle import cpu

    rng = np.random.default_rng(M + K + N)
    X = bf16_round(rng.standard_normal((M, K)) * 3 + 1.5)  # nonzero mean exercises the rank-1 correction
    Yt = bf16_round(rng.standard_normal((N, K)))
    ref = cpu.layernorm_matmul(X, Yt)
    assert_bf16_close(_run(torch, ops, X, Yt, torch.bfloat16), ref, f"K2 {M}x{K}x{N}")
    assert_f32_close(_run(torch, ops, X, Yt, torch.float32), ref, f"K2 fp32 {M}x{K}x{N}")


def test_c4_shape_properties(torch_ops):
    """C4 (M=65536, K=N=4096): sampled rows vs the oracle; O(2X) == O(X) bitwise
    (mean and variance scale exactly by powers of two)."""
    torch, ops = torch_ops
    from oracle import cpu

    g = torch.Generator(device="cuda").manual_seed(3)
    M, K, N = 65536, 4096, 4096
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    Yt = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    O = ops.layernorm_matmul(X, Yt)
    O2 = ops.layernorm_matmul(X * 2, Yt)
    torch.cuda.synchronize()
    assert torch.equal(O, O2)
    rows = torch.tensor([0, 127, 128, 30000, 65535], device="cuda")
    ref = cpu.layernorm_matmul(X[rows].double().cpu().numpy(), Yt.double().cpu().numpy())
    assert_bf16_close(O[rows].double().cpu().numpy(), ref, "K2 C4 sampled rows")
