"""Parity at every BASELINE.json configuration, at full shape, on every row and head.

Each config's output is compared element by element with a torch fp32 reference
computed on the device from the same bf16 inputs (tests/torch_ref.py), and on
stratified rows (one per 256-row m-unit, so every m-unit, scheduling group,
raster block and the last ragged unit is hit) with the float64 oracle
(oracle/bf_oracle.c, pinned to the reference build). These run the default
paths the planner picks at those shapes: C5 runs the wave sync with 2048-row
groups, C3 the segment sync with 4096-row groups, both on the CTA-pair kernel.
Tolerances are the north star's (tests/helpers.py). Mirrors the reference's
acceptance criteria (tests/acceptance.cpp:114-201) at the benchmark shapes.
"""
import numpy as np
import pytest

import torch_ref
from helpers import DeviceErr, assert_bf16_close, assert_f32_close, stratified_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_ops():
    import torch

    from paper_2505_07829_b200 import ops

    return torch, ops


def _ffn_inputs(torch, M, D, F, N, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    X = torch.randn(M, D, device="cuda", generator=g).bfloat16()
    Wt = torch.randn(F, D, device="cuda", generator=g).mul_(D ** -0.5).bfloat16()
    Vt = torch.randn(F, D, device="cuda", generator=g).mul_(D ** -0.5).bfloat16()
    Ut = torch.randn(N, F, device="cuda", generator=g).mul_(F ** -0.5).bfloat16()
    return X, Wt, Vt, Ut


def _check_ffn(torch, ops, M, D, F, N, seed, schedules=("fused",), oracle_unit=256):
    from oracle import cpu

    X, Wt, Vt, Ut = _ffn_inputs(torch, M, D, F, N, seed)
    outs = {s: ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule=s) for s in schedules}
    torch.cuda.synchronize()
    errs = {s: DeviceErr() for s in schedules}
    for rows, ref in torch_ref.rms_ffn_swiglu_chunks(X, Wt, Vt, Ut):
        for s in schedules:
            errs[s].add(outs[s][rows], ref)
    for s in schedules:
        errs[s].check(f"K1 {s} {M}x{D}x{F}x{N} all rows vs torch fp32")
    rows = stratified_rows(M, oracle_unit, seed)
    ref = cpu.rms_ffn_swiglu(X[rows].double().cpu().numpy(), Wt.double().cpu().numpy(), Vt.double().cpu().numpy(),
                             Ut.double().cpu().numpy())
    for s in schedules:
        assert_bf16_close(outs[s][rows].double().cpu().numpy(), ref, f"K1 {s} {M} rows, one per m-unit, vs oracle")
    return outs


def test_c3_every_row(torch_ops):
    """C3: Llama-3-8B FFN, 8192 tokens; fused (segment sync, 4096-row groups) and two-phase."""
    torch, ops = torch_ops
    plan = ops.plan("rms_ffn_swiglu", (8192, 4096, 14336, 4096))
    assert plan["kernel"] == "ffn_swiglu_2sm_kernel" and plan["sync"] == "segment" and plan["group"] * 256 == 4096
    _check_ffn(torch, ops, 8192, 4096, 14336, 4096, seed=11, schedules=("fused", "two_phase"))


def test_c5_every_row(torch_ops):
    """C5: Llama-3-70B FFN, 32768 tokens, the default >=1e13-FLOP path (wave sync, 2048-row groups)."""
    torch, ops = torch_ops
    plan = ops.plan("rms_ffn_swiglu", (32768, 8192, 28672, 8192))
    assert plan["sync"] == "wave" and plan["group"] * 256 == 2048 and plan["raster"] == 8, plan
    _check_ffn(torch, ops, 32768, 8192, 28672, 8192, seed=12)


def test_c5_shard_rows(torch_ops):
    """The 8-GPU shard of C5 (4096 rows) and of C3 (1024 rows): the strong-scaling launch sizes."""
    torch, ops = torch_ops
    _check_ffn(torch, ops, 4096, 8192, 28672, 8192, seed=13)
    _check_ffn(torch, ops, 1024, 4096, 14336, 4096, seed=14, schedules=("fused", "two_phase"))


@pytest.mark.parametrize("M", [7700, 8191])
def test_ragged_last_unit(torch_ops, M):
    """A ragged last m-unit at the C3 shape. M = 7700 is the size where the counter region of the
    workspace used to be one int short for the CTA-pair kernel (advice r01)."""
    torch, ops = torch_ops
    _check_ffn(torch, ops, M, 4096, 14336, 4096, seed=M, schedules=("fused", "two_phase"), oracle_unit=512)


def test_c4_every_row(torch_ops):
    """C4: LayerNorm->MatMul M=65536, K=N=4096."""
    torch, ops = torch_ops
    from oracle import cpu

    g = torch.Generator(device="cuda").manual_seed(21)
    M, K, N = 65536, 4096, 4096
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    Yt = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    O = ops.layernorm_matmul(X, Yt)
    torch.cuda.synchronize()
    err = DeviceErr()
    for rows, ref in torch_ref.layernorm_matmul_chunks(X, Yt):
        err.add(O[rows], ref)
    err.check("K2 C4 all rows vs torch fp32")
    rows = stratified_rows(M, 256, 21)
    ref = cpu.layernorm_matmul(X[rows].double().cpu().numpy(), Yt.double().cpu().numpy())
    assert_bf16_close(O[rows].double().cpu().numpy(), ref, "K2 C4 one row per m-unit vs oracle")


@pytest.mark.parametrize("ratio", [10.0, 100.0])
def test_lnmm_offset_mean_bf16(torch_ops, ratio):
    """Rows with |mu|/sigma = 10 and 100 (the GEMM runs on raw X with a rank-1 correction, and
    var = E[x^2] - mu^2). bf16 cannot hold a row with |mu|/sigma much above 100 (its spacing
    at |mu| is then sigma or more), so the bf16 mode stops here; see the fp32 cases below."""
    torch, ops = torch_ops
    from oracle import cpu

    from helpers import bf16_round

    rng = np.random.default_rng(int(ratio))
    M, K, N = 1024, 4096, 1024
    sign = np.where(rng.random((M, 1)) < 0.5, -1.0, 1.0)
    X = bf16_round(sign * ratio + rng.standard_normal((M, K)))
    Yt = bf16_round(rng.standard_normal((N, K)))
    x = torch.from_numpy(X).cuda().bfloat16()
    y = torch.from_numpy(Yt).cuda().bfloat16()
    out = ops.layernorm_matmul(x, y)
    torch.cuda.synchronize()
    assert_bf16_close(out.double().cpu().numpy(), cpu.layernorm_matmul(X, Yt), f"K2 bf16 |mu|/sigma={ratio}")


@pytest.mark.parametrize("ratio", [1e2, 1e3, 1e4])
def test_lnmm_offset_mean_fp32(torch_ops, ratio):
    """fp32 mode with |mu|/sigma up to 1e4 at the 1e-4 bar: the fp32 kernel shifts each row by a
    pivot (its first element) before both the statistics and the contraction, so neither
    var = E[x^2] - mu^2 nor X Yt^T - mu colsum(Yt) cancels catastrophically."""
    torch, ops = torch_ops
    from oracle import cpu

    rng = np.random.default_rng(int(ratio) + 1)
    M, K, N = 256, 1024, 256
    X = (ratio + rng.standard_normal((M, K))).astype(np.float32).astype(np.float64)
    Yt = rng.standard_normal((N, K)).astype(np.float32).astype(np.float64)
    out = ops.layernorm_matmul(torch.from_numpy(X).cuda().float(), torch.from_numpy(Yt).cuda().float())
    torch.cuda.synchronize()
    assert_f32_close(out.double().cpu().numpy(), cpu.layernorm_matmul(X, Yt), f"K2 fp32 |mu|/sigma={ratio:g}")


def test_c2_every_head(torch_ops):
    """C2: attention B=8, H=32, S=2048, D=128, all 256 heads; oracle on two query rows per
    256-row query tile of every head."""
    torch, ops = torch_ops
    from oracle import cpu

    g = torch.Generator(device="cuda").manual_seed(31)
    B, H, S, D = 8, 32, 2048, 128
    Q = torch.randn(B, H, S, D, device="cuda", generator=g).bfloat16()
    K = torch.randn(B, H, S, D, device="cuda", generator=g).bfloat16()
    Vt = torch.randn(B, H, D, S, device="cuda", generator=g).bfloat16()
    O = ops.attention(Q, K, Vt)
    torch.cuda.synchronize()
    err = DeviceErr()
    Of = O.reshape(B * H, S, D)
    for heads, ref in torch_ref.attention_chunks(Q, K, Vt):
        err.add(Of[heads], ref)
    # attention outputs are averages: rms(O) << rms(V), the normalized bar is 2e-2 (test_attention_gpu.py)
    err.check("K3 C2 all heads vs torch fp32", norm_tol=2e-2)
    rows = np.concatenate([stratified_rows(S, 256, 31), stratified_rows(S, 128, 32)[1::2]])
    q = Q.reshape(B * H, S, D)[:, rows].double().cpu().numpy()
    ref = cpu.attention_safe(q, K.reshape(B * H, S, D).double().cpu().numpy(),
                             Vt.reshape(B * H, D, S).double().cpu().numpy())
    assert_bf16_close(Of[:, rows].double().cpu().numpy(), ref, "K3 C2 every head, stratified rows vs oracle",
                      norm_tol=2e-2)


def test_c1_every_row_fp32(torch_ops):
    """C1: M=K=N=1024 fp32, all rows vs the float64 oracle at the 1e-4 bar."""
    torch, ops = torch_ops
    from oracle import cpu

    rng = np.random.default_rng(2001)
    X = rng.standard_normal((1024, 1024)).astype(np.float32).astype(np.float64)
    Yt = rng.standard_normal((1024, 1024)).astype(np.float32).astype(np.float64)
    out = ops.layernorm_matmul(torch.from_numpy(X).cuda().float(), torch.from_numpy(Yt).cuda().float())
    torch.cuda.synchronize()
    assert_f32_close(out.double().cpu().numpy(), cpu.layernorm_matmul(X, Yt), "C1 fp32 all rows")


def test_c3_fp32_tensor_cores(torch_ops):
    """K1 fp32 mode at the C3 shape (3xTF32 on tcgen05: split launch, gate/up GEMM with the SwiGLU
    epilogue writing h as hi/lo, down GEMM): one row per 128-row m-tile plus the last row vs the
    float64 oracle at the 1e-4 bar (contractions of 4096 and 14336)."""
    torch, ops = torch_ops
    from oracle import cpu

    M, D, F, N = 8192, 4096, 14336, 4096
    plan = ops.plan("rms_ffn_swiglu", (M, D, F, N), dtype=torch.float32)
    assert plan["kernel"] == "f32x3_gemm_kernel<gate>", plan
    g = torch.Generator(device="cuda").manual_seed(41)
    X = torch.randn(M, D, device="cuda", generator=g)
    Wt = torch.randn(F, D, device="cuda", generator=g) * D ** -0.5
    Vt = torch.randn(F, D, device="cuda", generator=g) * D ** -0.5
    Ut = torch.randn(N, F, device="cuda", generator=g) * F ** -0.5
    O = ops.rms_ffn_swiglu(X, Wt, Vt, Ut)
    torch.cuda.synchronize()
    rows = np.append(stratified_rows(M, 128, 41), M - 1)
    ref = cpu.rms_ffn_swiglu(X[rows].double().cpu().numpy(), Wt.double().cpu().numpy(), Vt.double().cpu().numpy(),
                             Ut.double().cpu().numpy())
    assert_f32_close(O[rows].double().cpu().numpy(), ref, "K1 fp32 C3, one row per m-tile, vs oracle")


def test_c2_fp32_every_head(torch_ops):
    """K3 fp32 mode at the C2 shape (3xTF32 flash attention on tcgen05): every head on two query
    rows per 64-row block vs float64 on the device, at the 1e-4 bar."""
    torch, ops = torch_ops
    assert ops.plan("attention", (256, 2048, 2048, 128, 128), dtype=torch.float32)["kernel"] == "attn_f32x3_kernel"
    g = torch.Generator(device="cuda").manual_seed(42)
    BH, S, D = 256, 2048, 128
    Q = torch.randn(BH, S, D, device="cuda", generator=g)
    K = torch.randn(BH, S, D, device="cuda", generator=g)
    Vt = torch.randn(BH, D, S, device="cuda", generator=g)
    O = ops.attention(Q, K, Vt)
    torch.cuda.synchronize()
    rows = torch.from_numpy(np.concatenate([stratified_rows(S, 64, 42), stratified_rows(S, 64, 43)])).cuda()
    md = mr = 0.0
    for h0 in range(0, BH, 32):
        q = Q[h0:h0 + 32, rows].double()
        ref = torch.softmax(q @ K[h0:h0 + 32].double().transpose(1, 2) / D ** 0.5, -1) @ \
            Vt[h0:h0 + 32].double().transpose(1, 2)
        md = max(md, float((O[h0:h0 + 32, rows].double() - ref).abs().max()))
        mr = max(mr, float(ref.abs().max()))
    from helpers import F32_REL_TOL
    assert md / mr <= F32_REL_TOL, f"K3 fp32 C2: max|d|/max|ref| = {md / mr:.3e}"
