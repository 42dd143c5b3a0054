"""Every fusion snapshot has its own GPU plan.

The reference's driver returns one snapshot per fusion fixpoint (engine.hpp:45-56, 164) and
its tests check that every snapshot computes the unfused program's result
(tests/test_engine.cpp:102-109, 126-131, 149-154, 170-181). Here each snapshot runs as a
distinct launch plan and must match the float64 oracle:

  K2 snapshot 0: the row-statistics map (forall m: for k: sum x, sum x^2) as its own launch,
                 then the GEMM map (BF_SCHED_STAGED);
  K3 snapshot 0: P = exp(S) buffered in HBM (internal buffered edge T1) between a scores launch
                 and a P.Vt launch, with the exponent bases of safe_attention_rows
                 (safe_numerics.hpp:147-175) resolved before the second map;
  K1 snapshot 0: H in HBM between two launches (tests/test_ffn_gpu.py covers it).
"""
import numpy as np
import pytest

from helpers import assert_bf16_close, bf16_round

pytestmark = pytest.mark.gpu

ATTN_NORM_TOL = 2e-2  # as tests/test_attention_gpu.py: P's bf16 rounding scales with |V|


@pytest.fixture(scope="module")
def torch_ops():
    import torch

    from paper_2505_07829_b200 import ops

    return torch, ops


def _t(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()


@pytest.mark.parametrize("M,K,N", [(256, 256, 256), (700, 384, 520), (1000, 1024, 264)])
def test_lnmm_staged_matches_oracle_and_fused(torch_ops, M, K, N):
    torch, ops = torch_ops
    from oracle import cpu

    rng = np.random.default_rng(M + K + N)
    X = bf16_round(rng.standard_normal((M, K)) * 1.5 + 0.7)
    Yt = bf16_round(rng.standard_normal((N, K)))
    x, yt = _t(torch, X), _t(torch, Yt)
    staged = ops.layernorm_matmul(x, yt, schedule="staged")
    fused = ops.layernorm_matmul(x, yt)
    torch.cuda.synchronize()
    ref = cpu.layernorm_matmul(X, Yt)
    assert_bf16_close(staged.double().cpu().numpy(), ref, f"K2 staged {M}x{K}x{N}")
    # the two plans compute the same statistics with the same per-row reduction order
    d = (staged.float() - fused.float()).abs().max().item()
    assert d <= 2 ** -7 * fused.float().abs().max().item(), f"staged vs fused max|d| = {d}"
    assert ops.plan("layernorm_matmul", (M, K, N), schedule="staged")["schedule"] == "staged"


ATTN_CASES = [
    (2, 128, 128, 128, 128),
    (3, 300, 520, 128, 128),  # ragged queries and keys (Skv % 128 != 0)
    (2, 256, 1024, 64, 128),
    (2, 200, 384, 128, 64),
    (1, 128, 8, 64, 64),
]


@pytest.mark.parametrize("BH,Sq,Skv,D,Dv", ATTN_CASES)
def test_attention_staged_matches_oracle(torch_ops, BH, Sq, Skv, D, Dv):
    torch, ops = torch_ops
    from oracle import cpu

    rng = np.random.default_rng(BH * 7 + Sq + Skv + D + Dv)
    Q = bf16_round(rng.standard_normal((BH, Sq, D)))
    K = bf16_round(rng.standard_normal((BH, Skv, D)))
    Vt = bf16_round(rng.standard_normal((BH, Dv, Skv)))
    out = ops.attention(_t(torch, Q), _t(torch, K), _t(torch, Vt), schedule="staged")
    torch.cuda.synchronize()
    ref = cpu.attention_safe(Q, K, Vt)
    assert_bf16_close(out.double().cpu().numpy(), ref, f"K3 staged {BH}x{Sq}x{Skv}x{D}x{Dv}", norm_tol=ATTN_NORM_TOL)


def test_attention_staged_rebases_written_blocks(torch_ops):
    """Logits that grow block after block (each key block's maximum exceeds the previous base by
    far more than 2^8): every written block of P must be rescaled to the final base, and large
    logits must stay finite (tests/test_safe_numerics.cpp:191-210)."""
    torch, ops = torch_ops
    from oracle import cpu

    rng = np.random.default_rng(5)
    BH, Sq, Skv, D = 2, 256, 768, 128
    Q = bf16_round(rng.standard_normal((BH, Sq, D)) * 0.5)
    K = rng.standard_normal((BH, Skv, D)) * 0.5
    # key block j gets an offset along Q's mean direction, so block maxima climb with j
    K += (np.arange(Skv) // 128)[None, :, None] * 3.0 * np.sign(Q.mean(axis=1, keepdims=True))
    K = bf16_round(K)
    Vt = bf16_round(rng.standard_normal((BH, D, Skv)))
    out = ops.attention(_t(torch, Q), _t(torch, K), _t(torch, Vt), schedule="staged")
    fused = ops.attention(_t(torch, Q), _t(torch, K), _t(torch, Vt))
    torch.cuda.synchronize()
    ref = cpu.attention_safe(Q, K, Vt)
    assert_bf16_close(out.double().cpu().numpy(), ref, "K3 staged, climbing logits", norm_tol=ATTN_NORM_TOL)
    assert_bf16_close(fused.double().cpu().numpy(), ref, "K3 fused, climbing logits", norm_tol=ATTN_NORM_TOL)


def test_attention_staged_c2_heads(torch_ops):
    """C2's shape (S=2048, D=128) on 8 heads: staged vs the fused kernel and the oracle on sampled rows."""
    torch, ops = torch_ops
    from oracle import cpu

    g = torch.Generator(device="cuda").manual_seed(3)
    BH, S, D = 8, 2048, 128
    Q = torch.randn(BH, S, D, device="cuda", generator=g).bfloat16()
    K = torch.randn(BH, S, D, device="cuda", generator=g).bfloat16()
    Vt = torch.randn(BH, D, S, device="cuda", generator=g).bfloat16()
    staged = ops.attention(Q, K, Vt, schedule="staged")
    fused = ops.attention(Q, K, Vt)
    torch.cuda.synchronize()
    d = (staged.float() - fused.float()).abs().max().item()
    assert d <= 2e-2 * fused.float().abs().max().item(), f"staged vs fused max|d| = {d}"
    rows = np.arange(0, S, 97)
    ref = cpu.attention_safe(Q[:, rows].double().cpu().numpy(), K.double().cpu().numpy(), Vt.double().cpu().numpy())
    assert_bf16_close(staged[:, rows].double().cpu().numpy(), ref, "K3 staged C2 rows", norm_tol=ATTN_NORM_TOL)
    plan = ops.plan("attention", (BH, S, S, D, D), schedule="staged")
    assert plan["schedule"] == "staged" and "attn_pv_kernel" in plan["kernel"]
