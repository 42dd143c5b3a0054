"""The planner's choice among the fp32-mode kernels, and each choice's parity at a small shape.

fp32 inputs must match the float64 reference within 1e-4 (tests/helpers.py). The default plans
are the 3xTF32 tensor-core kernels; K3 falls back to the FP32 FMA flash attention when the key
length is not a multiple of 4 (the TMA row pitch), and to the generic FMA kernel for head dims
other than 64/128."""
import numpy as np
import pytest

from helpers import assert_f32_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_ops():
    import torch

    from paper_2505_07829_b200 import ops

    return torch, ops


@pytest.mark.parametrize("dims,kernel", [
    ((2, 130, 256, 128, 128), "attn_f32x3_kernel"),
    ((2, 130, 64, 64, 64), "attn_f32x3_kernel"),
    ((2, 130, 250, 128, 64), "attn_f32_tiled_kernel"),  # Skv % 4 != 0
    ((2, 130, 256, 96, 80), "attn_f32_kernel"),  # head dims outside 64/128
])
def test_attention_fp32_plan_and_parity(torch_ops, dims, kernel):
    torch, ops = torch_ops
    from oracle import cpu

    BH, Sq, Skv, D, Dv = dims
    assert ops.plan("attention", dims, dtype=torch.float32)["kernel"] == kernel
    rng = np.random.default_rng(sum(dims))
    Q = rng.standard_normal((BH, Sq, D)).astype(np.float32).astype(np.float64)
    K = rng.standard_normal((BH, Skv, D)).astype(np.float32).astype(np.float64)
    Vt = rng.standard_normal((BH, Dv, Skv)).astype(np.float32).astype(np.float64)
    f = lambda a: torch.from_numpy(a).cuda().float()  # noqa: E731
    out = ops.attention(f(Q), f(K), f(Vt))
    torch.cuda.synchronize()
    assert_f32_close(out.double().cpu().numpy(), cpu.attention_safe(Q, K, Vt), f"K3 fp32 {kernel} {dims}")


def test_ffn_and_lnmm_fp32_plans(torch_ops):
    torch, ops = torch_ops
    assert ops.plan("rms_ffn_swiglu", (300, 256, 520, 136), dtype=torch.float32)["kernel"] == "f32x3_gemm_kernel<gate>"
    assert ops.plan("layernorm_matmul", (300, 256, 136), dtype=torch.float32)["kernel"] == "f32x3_gemm_kernel"


def test_attention_fp32_large_scores(torch_ops):
    """Scores spread over many octaves (|q| ~ 8): the 2^8 lazy rebase fires on many rows and
    blocks, and the warp-collective rescale of O in TMEM runs with mixed lanes."""
    torch, ops = torch_ops
    from oracle import cpu

    rng = np.random.default_rng(5)
    Q = (rng.standard_normal((2, 256, 64)) * 8).astype(np.float32).astype(np.float64)
    K = rng.standard_normal((2, 1024, 64)).astype(np.float32).astype(np.float64)
    Vt = rng.standard_normal((2, 64, 1024)).astype(np.float32).astype(np.float64)
    f = lambda a: torch.from_numpy(a).cuda().float()  # noqa: E731
    out = ops.attention(f(Q), f(K), f(Vt))
    torch.cuda.synchronize()
    assert_f32_close(out.double().cpu().numpy(), cpu.attention_safe(Q, K, Vt), "K3 fp32 large scores")
