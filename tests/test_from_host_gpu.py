"""ops.from_host: the host-buffer call shape of the reference's execute() (inputs and output in
pinned host memory), copies overlapped with the kernels in row slices. Rows (heads for
attention) are independent in every block program, so the sliced result must equal the
single device-resident call bit for bit."""
import pytest
import torch

from paper_2505_07829_b200 import ops

pytestmark = pytest.mark.gpu


def _pinned(t):
    return t.cpu().pin_memory()


@pytest.mark.parametrize("chunks", [1, 3, 4])
def test_ffn_from_host_matches_device(chunks):
    g = torch.Generator(device="cuda").manual_seed(1)
    M, D, F = 1000, 512, 768
    X = torch.randn(M, D, device="cuda", generator=g).bfloat16()
    Wt, Vt = [(torch.randn(F, D, device="cuda", generator=g) / 16).bfloat16() for _ in range(2)]
    Ut = (torch.randn(D, F, device="cuda", generator=g) / 16).bfloat16()
    for sched in ("fused", "two_phase"):
        ref = ops.rms_ffn_swiglu(X, Wt, Vt, Ut, schedule=sched)
        out = torch.empty(M, D, dtype=torch.bfloat16).pin_memory()
        ops.from_host(ops.rms_ffn_swiglu, [_pinned(X)], [_pinned(Wt), _pinned(Vt), _pinned(Ut)], out, chunks=chunks,
                      schedule=sched)
        torch.cuda.synchronize()
        assert torch.equal(out, ref.cpu()), sched


def test_lnmm_and_attention_from_host_match_device():
    g = torch.Generator(device="cuda").manual_seed(2)
    X = torch.randn(700, 384, device="cuda", generator=g).bfloat16()
    Yt = torch.randn(256, 384, device="cuda", generator=g).bfloat16()
    ref = ops.layernorm_matmul(X, Yt)
    out = torch.empty(700, 256, dtype=torch.bfloat16).pin_memory()
    ops.from_host(ops.layernorm_matmul, [_pinned(X)], [_pinned(Yt)], out, chunks=3)
    torch.cuda.synchronize()
    assert torch.equal(out, ref.cpu())

    Q = torch.randn(6, 4, 300, 128, device="cuda", generator=g).bfloat16()
    K = torch.randn(6, 4, 256, 128, device="cuda", generator=g).bfloat16()
    Vt = torch.randn(6, 4, 128, 256, device="cuda", generator=g).bfloat16()
    ref = ops.attention(Q, K, Vt)
    out = torch.empty(6, 4, 300, 128, dtype=torch.bfloat16).pin_memory()
    ops.from_host(ops.attention, [_pinned(Q), _pinned(K), _pinned(Vt)], [], out, chunks=4)
    torch.cuda.synchronize()
    assert torch.equal(out, ref.cpu())


def test_from_host_rejects_device_tensors():
    X = torch.zeros(4, 4, device="cuda")
    with pytest.raises(ValueError, match="host tensors"):
        ops.from_host(ops.layernorm_matmul, [X], [], torch.zeros(4, 4))


def test_back_to_back_calls_alternate_buffers_safely():
    """Consecutive calls reuse two device buffer sets; each call's output must be its own."""
    g = torch.Generator(device="cuda").manual_seed(3)
    M, K, N = 640, 256, 384
    Yt = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    Xs = [torch.randn(M, K, device="cuda", generator=g).bfloat16() for _ in range(5)]
    refs = [ops.layernorm_matmul(X, Yt).cpu() for X in Xs]
    hosts = [_pinned(X) for X in Xs]
    Yh = _pinned(Yt)
    outs = [torch.empty(M, N, dtype=torch.bfloat16).pin_memory() for _ in Xs]
    for Xh, o in zip(hosts, outs):
        ops.from_host(ops.layernorm_matmul, [Xh], [Yh], o, chunks=3)
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert torch.equal(o, r)
    ops.clear_host_buffers()
    o = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
    ops.from_host(ops.layernorm_matmul, [hosts[0]], [Yh], o, chunks=2)
    torch.cuda.synchronize()
    assert torch.equal(o, refs[0])
