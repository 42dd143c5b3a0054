"""The product calls inside CUDA graphs: serving stacks capture their forward passes, so each
plan (K1 fused and two-phase, K2 fused and staged, K3 fused and staged, fp32 K2) must be
capturable on a side stream and replay bit-identically to the eager call, with the replay
seeing new input values written into the same buffers (no value is baked in at capture).
"""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_ops():
    import torch

    from paper_2505_07829_b200 import ops

    return torch, ops


def _inputs(torch, kind, dtype):
    g = torch.Generator(device="cuda").manual_seed(5)
    r = lambda *s: torch.randn(*s, device="cuda", generator=g).to(dtype)  # noqa: E731
    if kind == "ffn":
        return [r(700, 256), r(384, 256) * 0.06, r(384, 256) * 0.06, r(264, 384) * 0.05]
    if kind == "lnmm":
        return [r(900, 320) + 1.0, r(264, 320)]
    return [r(3, 300, 128), r(3, 456, 128), r(3, 128, 456)]


CASES = [("ffn", "fused", "bf16"), ("ffn", "two_phase", "bf16"), ("lnmm", "fused", "bf16"),
         ("lnmm", "staged", "bf16"), ("lnmm", "fused", "f32"), ("attn", "fused", "bf16"),
         ("attn", "staged", "bf16")]


@pytest.mark.parametrize("kind,schedule,dt", CASES)
def test_capture_and_replay(torch_ops, kind, schedule, dt):
    torch, ops = torch_ops
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    fn = {"ffn": ops.rms_ffn_swiglu, "lnmm": ops.layernorm_matmul, "attn": ops.attention}[kind]
    args = _inputs(torch, kind, dtype)
    eager = fn(*args, schedule=schedule)
    torch.cuda.synchronize()
    out = torch.empty_like(eager)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(*args, schedule=schedule, out=out)  # warm the plan and workspace caches on this stream
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        fn(*args, schedule=schedule, out=out)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager), f"{kind} {schedule} {dt}: graph replay differs from the eager call"
    # new values in the captured input buffers: the replay must compute on them
    args[0].copy_(args[0] * 0.5 + 0.25)
    eager2 = fn(*args, schedule=schedule)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager2) and not torch.equal(eager2, eager)
