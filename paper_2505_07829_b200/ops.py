"""Torch-tensor front end over the C-ABI (device memory and streams only).

PyTorch is plumbing here: it owns the device buffers and the current stream.
All arithmetic happens in libbfgpu.so kernels. Every function validates
shapes/dtypes and raises BfError with the library's message on failure.
"""
from __future__ import annotations

import torch

from . import _lib
from ._lib import (BF_DTYPE_BF16, BF_DTYPE_F32, BF_PATTERN_ATTENTION, BF_PATTERN_LAYERNORM_MATMUL,
                   BF_PATTERN_RMS_FFN_SWIGLU, BF_SCHED_FUSED, BF_SCHED_STAGED, check)

# schedule name -> code. "two_phase" (the first fusion snapshot of each program) is the name the
# K1 API has always used; "staged" is the same thing.
SCHEDULES = {"fused": BF_SCHED_FUSED, "two_phase": BF_SCHED_STAGED, "staged": BF_SCHED_STAGED}

# one cached workspace per (device, stream): calls on different streams may overlap
_WS: dict[tuple[int, int], torch.Tensor] = {}


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return BF_DTYPE_BF16
    if t.dtype == torch.float32:
        return BF_DTYPE_F32
    raise TypeError(f"unsupported dtype {t.dtype}; expected bfloat16 or float32")


def _require(t: torch.Tensor, name: str, shape: tuple, dtype: torch.dtype, device) -> None:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.dtype != dtype:
        raise ValueError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (row-major)")


def _workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    key = (idx, _stream_ptr(device))
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def rms_ffn_swiglu(X, Wt, Vt, Ut, eps: float = 0.0, schedule: str = "fused", out=None, workspace=None):
    """O = (swish(r*X Wt^T) * (r*X Vt^T)) Ut^T with r = 1/sqrt(mean(X^2) + eps).

    Mirrors ref::rms_ffn_swiglu (interpreter.hpp:553-559): X[M,D], Wt/Vt[F,D],
    Ut[N,F] ("transposed" right operands, lowering.hpp:583-597).
    """
    M, D = X.shape
    F = Wt.shape[0]
    N = Ut.shape[0]
    dt = X.dtype
    dev = X.device
    _require(X, "X", (M, D), dt, dev)
    _require(Wt, "Wt", (F, D), dt, dev)
    _require(Vt, "Vt", (F, D), dt, dev)
    _require(Ut, "Ut", (N, F), dt, dev)
    sched = SCHEDULES[schedule]
    if out is None:
        out = torch.empty((M, N), dtype=dt, device=dev)
    _require(out, "out", (M, N), dt, dev)
    code = _dtype_code(X)
    L = _lib.lib()
    nbytes = L.bf_rms_ffn_swiglu_workspace_bytes(M, D, F, N, code, sched)
    with torch.cuda.device(dev):  # the C-ABI launches on the current device
        ws = workspace if workspace is not None else _workspace(nbytes, dev)
        check(
            L.bf_rms_ffn_swiglu(
                X.data_ptr(), Wt.data_ptr(), Vt.data_ptr(), Ut.data_ptr(), out.data_ptr(), M, D, F, N, code,
                float(eps), sched, ws.data_ptr(), ws.numel(), _stream_ptr(dev),
            )
        )
    return out


def layernorm_matmul(X, Yt, eps: float = 0.0, out=None, workspace=None, schedule: str = "fused"):
    """O = layernorm(X) Yt^T without eps/gamma/beta (ref::layernorm_matmul, interpreter.hpp:549-551).

    schedule "fused": the final fusion snapshot (statistics inside the GEMM launch); "staged":
    the first snapshot (the row-statistics map as its own launch, then the GEMM map).
    """
    sched = SCHEDULES[schedule]
    M, K = X.shape
    N = Yt.shape[0]
    dt = X.dtype
    dev = X.device
    _require(X, "X", (M, K), dt, dev)
    _require(Yt, "Yt", (N, K), dt, dev)
    if out is None:
        out = torch.empty((M, N), dtype=dt, device=dev)
    _require(out, "out", (M, N), dt, dev)
    code = _dtype_code(X)
    L = _lib.lib()
    nbytes = L.bf_layernorm_matmul_workspace_bytes(M, K, N, code)
    with torch.cuda.device(dev):
        ws = workspace if workspace is not None else _workspace(nbytes, dev)
        check(
            L.bf_layernorm_matmul_sched(
                X.data_ptr(), Yt.data_ptr(), out.data_ptr(), M, K, N, code, float(eps), sched, ws.data_ptr(),
                ws.numel(), _stream_ptr(dev),
            )
        )
    return out


def attention(Q, K, Vt, scale: float | None = None, out=None, schedule: str = "fused", workspace=None):
    """O = softmax(scale Q K^T) V with V given as Vt (ref::attention, interpreter.hpp:543-547).

    Q: [..., Sq, D], K: [..., Skv, D], Vt: [..., Dv, Skv]; leading dims are heads.
    schedule "fused": the final snapshot (online softmax, P never leaves the chip); "staged":
    the first snapshot (P = exp(S) buffered in an HBM workspace between two launches; bf16).
    """
    sched = SCHEDULES[schedule]
    *lead, Sq, D = Q.shape
    Skv = K.shape[-2]
    Dv = Vt.shape[-2]
    BH = 1
    for x in lead:
        BH *= x
    dt = Q.dtype
    dev = Q.device
    _require(Q, "Q", (*lead, Sq, D), dt, dev)
    _require(K, "K", (*lead, Skv, D), dt, dev)
    _require(Vt, "Vt", (*lead, Dv, Skv), dt, dev)
    if out is None:
        out = torch.empty((*lead, Sq, Dv), dtype=dt, device=dev)
    _require(out, "out", (*lead, Sq, Dv), dt, dev)
    L = _lib.lib()
    code = _dtype_code(Q)
    nbytes = L.bf_attention_workspace_bytes(BH, Sq, Skv, D, Dv, code, sched)
    with torch.cuda.device(dev):
        ws_ptr, ws_len = 0, 0
        if nbytes:
            ws = workspace if workspace is not None else _workspace(nbytes, dev)
            ws_ptr, ws_len = ws.data_ptr(), ws.numel()
        check(
            L.bf_attention_sched(
                Q.data_ptr(), K.data_ptr(), Vt.data_ptr(), out.data_ptr(), BH, Sq, Skv, D, Dv, code,
                float(scale) if scale is not None else 0.0, sched, ws_ptr, ws_len, _stream_ptr(dev),
            )
        )
    return out


def kernel_launches() -> int:
    return int(_lib.lib().bf_kernel_launches())


def plan(pattern: str, dims, dtype=torch.bfloat16, schedule: str = "fused", device=None) -> dict:
    """The planner's launch plan (kernel, tiles, SMEM/TMEM budgets, grid, group, sync) for a call.

    pattern: "rms_ffn_swiglu" (dims M, D, F, N), "layernorm_matmul" (M, K, N) or
    "attention" (BH, Sq, Skv, D, Dv).
    """
    import ctypes
    import json

    pid = {"rms_ffn_swiglu": BF_PATTERN_RMS_FFN_SWIGLU, "layernorm_matmul": BF_PATTERN_LAYERNORM_MATMUL,
           "attention": BF_PATTERN_ATTENTION}[pattern]
    arr = (ctypes.c_int64 * len(dims))(*[int(d) for d in dims])
    buf = ctypes.create_string_buffer(8192)
    code = BF_DTYPE_BF16 if dtype == torch.bfloat16 else BF_DTYPE_F32
    sched = SCHEDULES[schedule]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.device(dev):
        check(_lib.lib().bf_plan_json(pid, arr, len(dims), code, sched, buf, len(buf)))
    return json.loads(buf.value.decode())


# ----------------------------------------------------------------- host-buffer calls
# The reference's execute() receives host matrices. from_host() is that call shape on the
# GPU: inputs in pinned host memory, output back into pinned host memory, with the copies
# overlapped with the kernels. Shared operands (weights) go first on an H2D stream; the
# row-sharded operands follow in `chunks` slices along dim 0 (rows, or heads for attention),
# each slice's kernel starts as soon as its slice has landed, and each slice's output
# leaves on a D2H stream while the next slice computes. Rows are independent in all three
# block programs (per-row statistics / per-head attention), so slicing is exact.
# Consecutive calls with the same shapes alternate between two sets of device buffers, so
# a call's host-to-device copies only wait for the kernels of the call before the previous
# one: back-to-back calls keep the H2D engine busy while the previous call computes.
_SIDE_STREAMS: dict[tuple[int, str], torch.cuda.Stream] = {}
_HOST_BUFS: dict[tuple, torch.Tensor] = {}
_SLOTS: dict[tuple, dict] = {}


def _side_stream(device: torch.device, name: str) -> torch.cuda.Stream:
    key = (device.index, name)
    s = _SIDE_STREAMS.get(key)
    if s is None:
        s = torch.cuda.Stream(device=device)
        _SIDE_STREAMS[key] = s
    return s


def _device_like(t: torch.Tensor, device: torch.device, tag: tuple) -> torch.Tensor:
    # keyed by the call signature and slot, never by shape alone: buffers are reused only by
    # calls whose slot events order them (two signatures with a same-shaped operand must not
    # share a buffer, or one call's H2D could overwrite it while the other's kernels read it)
    key = (device.index, tag)
    b = _HOST_BUFS.get(key)
    if b is None:
        b = torch.empty(t.shape, dtype=t.dtype, device=device)
        _HOST_BUFS[key] = b
    return b


def from_host(fn, row_inputs, shared_inputs, out_host, chunks: int = 4, **kwargs):
    """out_host = fn(*row_inputs, *shared_inputs) for pinned host tensors, copies overlapped.

    fn is one of rms_ffn_swiglu / layernorm_matmul / attention. Its row-sharded operands are
    `row_inputs` (sliced along dim 0), the rest `shared_inputs` (copied whole), in fn's
    argument order: row operands first. Returns out_host; the current stream is ordered
    after the last device-to-host copy.
    """
    for t in (*row_inputs, *shared_inputs, out_host):
        if t.is_cuda:
            raise ValueError("from_host takes host tensors")
    dev = torch.device("cuda", torch.cuda.current_device())
    comp = torch.cuda.current_stream(dev)
    h2d, d2h = _side_stream(dev, "h2d"), _side_stream(dev, "d2h")
    rows = row_inputs[0].shape[0]
    chunks = max(1, min(chunks, rows))
    bounds = [rows * k // chunks for k in range(chunks + 1)]
    sig = (dev.index, id(fn), tuple((tuple(t.shape), t.dtype) for t in (*row_inputs, *shared_inputs, out_host)))
    state = _SLOTS.setdefault(sig, {"next": 0, "computed": [None, None]})
    slot = state["next"]
    state["next"] ^= 1
    row_dev = [_device_like(t, dev, (sig, "row", i, slot)) for i, t in enumerate(row_inputs)]
    shared_dev = [_device_like(t, dev, (sig, "shared", i, slot)) for i, t in enumerate(shared_inputs)]
    out_dev = _device_like(out_host, dev, (sig, "out", 0, slot))
    if state["computed"][slot] is not None:
        h2d.wait_event(state["computed"][slot])  # kernels of the last call on this slot are done
    else:
        h2d.wait_stream(comp)
    ev_in = [torch.cuda.Event() for _ in range(chunks)]
    ev_out = [torch.cuda.Event() for _ in range(chunks)]
    with torch.cuda.stream(h2d):
        for h, d in zip(shared_inputs, shared_dev):
            d.copy_(h, non_blocking=True)
        for k in range(chunks):
            a, b = bounds[k], bounds[k + 1]
            for h, d in zip(row_inputs, row_dev):
                d[a:b].copy_(h[a:b], non_blocking=True)
            ev_in[k].record(h2d)
    for k in range(chunks):
        a, b = bounds[k], bounds[k + 1]
        comp.wait_event(ev_in[k])
        fn(*[d[a:b] for d in row_dev], *shared_dev, out=out_dev[a:b], **kwargs)
        ev_out[k].record(comp)
    computed = torch.cuda.Event()
    computed.record(comp)
    state["computed"][slot] = computed
    with torch.cuda.stream(d2h):
        for k in range(chunks):
            a, b = bounds[k], bounds[k + 1]
            d2h.wait_event(ev_out[k])
            out_host[a:b].copy_(out_dev[a:b], non_blocking=True)
    comp.wait_stream(d2h)
    return out_host


def clear_host_buffers() -> None:
    """Free the device buffers from_host() keeps per (shapes, dtypes) between calls."""
    torch.cuda.synchronize()
    _HOST_BUFS.clear()
    _SLOTS.clear()
