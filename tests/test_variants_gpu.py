"""Parity of the non-default kernel variants that the environment selects (read once per
process, hence the subprocesses): the 1-SM K1 and K2 kernels (BFGPU_FFN_1SM, BFGPU_LNMM_1SM),
the 512x256-tile K2 (BFGPU_LNMM_WIDE),
the FMA-pipe exponential splits of K3 (BFGPU_ATTN_EMU), non-default K1/K2 scheduling groups
(BFGPU_FFN_GROUP, BFGPU_LNMM_GROUP), the FP32 FMA kernels of the fp32 mode (BFGPU_F32_SIMT) and the K1 wave sync forced on at a size where it is off by default (BFGPU_FFN_WAVESYNC=1).
Same oracle and tolerances as the default-path tests."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SNIPPET = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from helpers import assert_bf16_close, assert_f32_close, bf16_round
from oracle import cpu
from paper_2505_07829_b200 import ops
rng = np.random.default_rng(7)
def t(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()
what = {what!r}
if what == "ffn":
    M, D, F, N = 520, 256, 392, 264
    X = bf16_round(rng.standard_normal((M, D))); Wt = bf16_round(rng.standard_normal((F, D)) / 16)
    Vt = bf16_round(rng.standard_normal((F, D)) / 16); Ut = bf16_round(rng.standard_normal((N, F)) / 16)
    for sched in ("fused", "two_phase"):
        out = ops.rms_ffn_swiglu(t(X), t(Wt), t(Vt), t(Ut), schedule=sched).double().cpu().numpy()
        assert_bf16_close(out, cpu.rms_ffn_swiglu(X, Wt, Vt, Ut), "K1 variant " + sched)
elif what == "lnmm":
    M, K, N = 600, 264, 392
    X = bf16_round(rng.standard_normal((M, K)) * 3 + 1.5); Yt = bf16_round(rng.standard_normal((N, K)))
    out = ops.layernorm_matmul(t(X), t(Yt)).double().cpu().numpy()
    assert_bf16_close(out, cpu.layernorm_matmul(X, Yt), "K2 variant")
elif what == "f32pair":
    # the CTA-pair 3xTF32 GEMMs (256 x 256 tiles, M = 256 MMAs) forced at ragged small shapes
    f = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().float()
    assert ops.plan("layernorm_matmul", (600, 264, 392), dtype=torch.float32)["kernel"].startswith("f32x3_pair")
    X = (rng.standard_normal((600, 264)) * 2 + 3).astype(np.float32).astype(np.float64)
    Y = rng.standard_normal((392, 264)).astype(np.float32).astype(np.float64)
    out = ops.layernorm_matmul(f(X), f(Y)).double().cpu().numpy()
    assert_f32_close(out, cpu.layernorm_matmul(X, Y), "K2 fp32 pair")
    X = rng.standard_normal((300, 136)).astype(np.float32).astype(np.float64)
    Wt = (rng.standard_normal((264, 136)) / 12).astype(np.float32).astype(np.float64)
    Vt = (rng.standard_normal((264, 136)) / 12).astype(np.float32).astype(np.float64)
    Ut = (rng.standard_normal((328, 264)) / 16).astype(np.float32).astype(np.float64)
    out = ops.rms_ffn_swiglu(f(X), f(Wt), f(Vt), f(Ut)).double().cpu().numpy()
    assert_f32_close(out, cpu.rms_ffn_swiglu(X, Wt, Vt, Ut), "K1 fp32 pair gate/up and down GEMMs")
elif what == "f32":
    # the FP32 FMA kernels (BFGPU_F32_SIMT=1) instead of the 3xTF32 tensor-core plans
    f = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().float()
    assert not ops.plan("attention", (3, 300, 456, 128, 64), dtype=torch.float32)["kernel"].startswith("attn_f32x3")
    X = rng.standard_normal((200, 136)).astype(np.float32).astype(np.float64)
    Wt = (rng.standard_normal((264, 136)) / 12).astype(np.float32).astype(np.float64)
    Vt = (rng.standard_normal((264, 136)) / 12).astype(np.float32).astype(np.float64)
    Ut = (rng.standard_normal((72, 264)) / 16).astype(np.float32).astype(np.float64)
    out = ops.rms_ffn_swiglu(f(X), f(Wt), f(Vt), f(Ut)).double().cpu().numpy()
    assert_f32_close(out, cpu.rms_ffn_swiglu(X, Wt, Vt, Ut), "K1 fp32 FMA")
    Y = rng.standard_normal((96, 136)).astype(np.float32).astype(np.float64)
    out = ops.layernorm_matmul(f(X), f(Y)).double().cpu().numpy()
    assert_f32_close(out, cpu.layernorm_matmul(X, Y), "K2 fp32 FMA")
    Q = rng.standard_normal((3, 300, 128)).astype(np.float32).astype(np.float64)
    K = rng.standard_normal((3, 456, 128)).astype(np.float32).astype(np.float64)
    Vt = rng.standard_normal((3, 64, 456)).astype(np.float32).astype(np.float64)
    out = ops.attention(f(Q), f(K), f(Vt)).double().cpu().numpy()
    assert_f32_close(out, cpu.attention_safe(Q, K, Vt), "K3 fp32 FMA")
else:
    Q = bf16_round(rng.standard_normal((3, 300, 128))); K = bf16_round(rng.standard_normal((3, 456, 128)))
    Vt = bf16_round(rng.standard_normal((3, 128, 456)))
    out = ops.attention(t(Q), t(K), t(Vt)).double().cpu().numpy()
    assert_bf16_close(out, cpu.attention_safe(Q, K, Vt), "K3 variant", norm_tol=2e-2)
print("ok")
"""


@pytest.mark.parametrize(
    "what,env",
    [
        ("ffn", {"BFGPU_FFN_1SM": "1"}),
        ("ffn", {"BFGPU_FFN_GROUP": "1"}),
        ("ffn", {"BFGPU_FFN_GROUP": "64"}),
        ("ffn", {"BFGPU_FFN_WAVESYNC": "1"}),
        ("ffn", {"BFGPU_FFN_SEGSYNC": "0"}),
        ("ffn", {"BFGPU_FFN_BRASTER": "0"}),
        ("ffn", {"BFGPU_FFN_BRASTER": "3"}),
        ("lnmm", {"BFGPU_LNMM_1SM": "1"}),
        ("lnmm", {"BFGPU_LNMM_GROUP": "2"}),
        ("lnmm", {"BFGPU_LNMM_WIDE": "1"}),
        ("attn", {"BFGPU_ATTN_EMU": "0"}),
        ("attn", {"BFGPU_ATTN_EMU": "12"}),
        ("attn", {"BFGPU_ATTN_EMU": "16"}),
        ("f32", {"BFGPU_F32_SIMT": "1"}),
        ("f32pair", {"BFGPU_F32_PAIR": "1", "BFGPU_F32_K1_PAIR": "1"}),
        ("f32pair", {"BFGPU_F32_PAIR": "1", "BFGPU_F32_K1_PAIR": "1", "BFGPU_F32_GROUP": "1"}),
    ],
)
def test_variant_matches_oracle(what, env):
    code = SNIPPET.format(root=str(ROOT), tests=str(ROOT / "tests"), what=what)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       env={**os.environ, **env})
    assert r.returncode == 0 and "ok" in r.stdout, f"{env}\n{r.stdout}\n{r.stderr[-3000:]}"
