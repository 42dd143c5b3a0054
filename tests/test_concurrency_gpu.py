"""Concurrent calls (the reference contract allows them: SPEC.md:440, interpreter.hpp:478-487).

K1 and K2 spin-wait on grid-wide counters, so they launch cooperatively (plan.hpp
launch_planned): the driver starts such a grid only when all of its CTAs can be resident. These
tests overlap the three programs on separate streams, and from separate host threads, and
require every result to be bit-identical to the same call made alone.
"""
import threading

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch

    from paper_2505_07829_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(11)

    def r(*shape, scale=1.0):
        return (torch.randn(*shape, device="cuda", generator=g) * scale).bfloat16()

    ffn = (r(2048, 1024), r(3072, 1024, scale=0.03), r(3072, 1024, scale=0.03), r(1024, 3072, scale=0.02))
    ln = (r(4096, 1024) * 2 + 1, r(1536, 1024))
    at = (r(16, 1024, 128), r(16, 1024, 128), r(16, 128, 1024))
    return torch, ops, ffn, ln, at


def _alone(torch, ops, ffn, ln, at):
    o1 = ops.rms_ffn_swiglu(*ffn)
    o2 = ops.layernorm_matmul(*ln)
    o3 = ops.attention(*at)
    torch.cuda.synchronize()
    return o1, o2, o3


def test_three_programs_on_three_streams(setup):
    torch, ops, ffn, ln, at = setup
    ref = _alone(torch, ops, ffn, ln, at)
    streams = [torch.cuda.Stream() for _ in range(3)]
    torch.cuda.synchronize()
    for _ in range(5):
        outs = [None] * 3
        # each stream gets its own workspace (ops caches one per (device, stream))
        with torch.cuda.stream(streams[0]):
            outs[0] = ops.rms_ffn_swiglu(*ffn)
        with torch.cuda.stream(streams[1]):
            outs[1] = ops.layernorm_matmul(*ln)
        with torch.cuda.stream(streams[2]):
            outs[2] = ops.attention(*at)
        torch.cuda.synchronize()
        for o, rf, name in zip(outs, ref, ("K1", "K2", "K3")):
            assert torch.equal(o, rf), f"{name} on a concurrent stream differs from the call made alone"


def test_two_host_threads(setup):
    """Two host threads, each on its own stream, calling K1 and K2 in a loop: per-thread error state
    and workspaces must not interfere."""
    torch, ops, ffn, ln, at = setup
    ref = _alone(torch, ops, ffn, ln, at)
    errors = []

    def worker(kind):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(6):
                    o = ops.rms_ffn_swiglu(*ffn) if kind == 0 else ops.layernorm_matmul(*ln)
                    s.synchronize()
                    if not torch.equal(o, ref[kind]):
                        errors.append(f"thread {kind}: result differs")
        except Exception as e:  # noqa: BLE001
            errors.append(f"thread {kind}: {e}")

    th = [threading.Thread(target=worker, args=(k,)) for k in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors


def test_error_is_per_thread(setup):
    """bf_last_error() is thread-local: a failing call on one thread does not overwrite another's."""
    torch, ops, ffn, ln, at = setup
    from paper_2505_07829_b200 import _lib

    L = _lib.lib()
    assert L.bf_attention(0, 0, 0, 0, 1, 128, 128, 128, 128, 0, 0.0, 0) != 0
    mine = L.bf_last_error().decode()
    assert "null" in mine
    other = {}

    def bad():
        rc = L.bf_layernorm_matmul(1, 1, 1, 0, 8, 8, 0, 0.0, 0, 0, 0)  # M = 0
        other["rc"], other["msg"] = rc, L.bf_last_error().decode()

    t = threading.Thread(target=bad)
    t.start()
    t.join()
    assert other["rc"] != 0 and other["msg"] and other["msg"] != mine
    assert L.bf_last_error().decode() == mine
