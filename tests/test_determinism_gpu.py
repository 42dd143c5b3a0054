"""Run-to-run determinism of every plan (the backend's side of the reference's acceptance
criterion 9, tests/acceptance.cpp:808-833): the same call on the same inputs gives the same
bits, with other work launched in between (so no result depends on timing, L2 contents or
scheduling order), and the program-file route verifies a snapshot against itself."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def torch_ops():
    import torch

    from paper_2505_07829_b200 import ops

    return torch, ops


def _inputs(torch, kind, dtype):
    g = torch.Generator(device="cuda").manual_seed(9)
    r = lambda *s: torch.randn(*s, device="cuda", generator=g).to(dtype)  # noqa: E731
    if kind == "ffn":
        return [r(1500, 512), r(768, 512) * 0.05, r(768, 512) * 0.05, r(520, 768) * 0.04]
    if kind == "lnmm":
        return [r(1800, 520) + 2.0, r(776, 520)]
    return [r(5, 700, 128), r(5, 904, 128), r(5, 128, 904) * 3.0]


CASES = [("ffn", "fused", "bf16"), ("ffn", "two_phase", "bf16"), ("ffn", "fused", "f32"),
         ("lnmm", "fused", "bf16"), ("lnmm", "staged", "bf16"), ("lnmm", "fused", "f32"),
         ("attn", "fused", "bf16"), ("attn", "staged", "bf16"), ("attn", "fused", "f32")]


@pytest.mark.parametrize("kind,schedule,dt", CASES)
def test_bitwise_repeatable(torch_ops, kind, schedule, dt):
    torch, ops = torch_ops
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    fn = {"ffn": ops.rms_ffn_swiglu, "lnmm": ops.layernorm_matmul, "attn": ops.attention}[kind]
    args = _inputs(torch, kind, dtype)
    first = fn(*args, schedule=schedule).clone()
    noise = torch.randn(4096, 4096, device="cuda")
    for _ in range(3):
        noise = noise @ noise.T * 1e-3  # unrelated work between the calls
        again = fn(*args, schedule=schedule)
        torch.cuda.synchronize()
        assert torch.equal(again, first), f"{kind} {schedule} {dt}: run-to-run difference"


def test_snapshot_verifies_against_itself():
    cli = ROOT / "paper_2505_07829_b200" / "lib" / "bfgpu-cli"
    if not cli.exists():
        pytest.skip("bfgpu-cli not built")
    snap = ROOT / "tests" / "golden" / "programs" / "layernorm-matmul" / "snapshot_2.json"
    r = subprocess.run([str(cli), "verify", str(snap), "--dims", "M=2,N=2,K=2", "--block", "4x4", "--trials", "3"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "verdict: equivalent" in r.stdout, r.stdout + r.stderr
