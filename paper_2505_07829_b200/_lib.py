"""ctypes binding of the C-ABI in include/bfgpu.h (libbfgpu.so, built in-tree).

This is the reference-side binding a Python caller would add; it is also what
the tests and bench.py use. It never falls back to anything: if the shared
library is missing the import of an op raises.
"""
from __future__ import annotations

import ctypes
import threading
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libbfgpu.so"
_lock = threading.Lock()
_lib = None

BF_OK = 0
BF_ERR_INVALID_ARGUMENT = 1
BF_ERR_UNSUPPORTED = 2
BF_ERR_CUDA = 3
BF_ERR_INTERNAL = 4

BF_DTYPE_BF16 = 0
BF_DTYPE_F32 = 1

BF_SCHED_FUSED = 0
BF_SCHED_STAGED = 1
BF_FFN_FUSED = BF_SCHED_FUSED
BF_FFN_TWO_PHASE = BF_SCHED_STAGED

BF_PATTERN_RMS_FFN_SWIGLU = 0
BF_PATTERN_LAYERNORM_MATMUL = 1
BF_PATTERN_ATTENTION = 2

# (name, restype, argtypes) for every symbol declared in include/bfgpu.h
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_SIGNATURES = [
    ("bf_rms_ffn_swiglu_workspace_bytes", ctypes.c_size_t, [_i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int]),
    (
        "bf_rms_ffn_swiglu",
        ctypes.c_int,
        [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_float, ctypes.c_int, _vp,
         ctypes.c_size_t, _vp],
    ),
    ("bf_layernorm_matmul_workspace_bytes", ctypes.c_size_t, [_i64, _i64, _i64, ctypes.c_int]),
    (
        "bf_layernorm_matmul",
        ctypes.c_int,
        [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, ctypes.c_float, _vp, ctypes.c_size_t, _vp],
    ),
    (
        "bf_layernorm_matmul_sched",
        ctypes.c_int,
        [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, ctypes.c_float, ctypes.c_int, _vp, ctypes.c_size_t, _vp],
    ),
    (
        "bf_attention",
        ctypes.c_int,
        [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_float, _vp],
    ),
    ("bf_attention_workspace_bytes", ctypes.c_size_t, [_i64, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int]),
    (
        "bf_attention_sched",
        ctypes.c_int,
        [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_float, ctypes.c_int, _vp,
         ctypes.c_size_t, _vp],
    ),
    ("bf_jit_compile", ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_vp), ctypes.c_char_p, ctypes.c_size_t]),
    ("bf_jit_check", ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t]),
    ("bf_jit_launch", ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint,
                                     ctypes.c_size_t, _vp, ctypes.POINTER(_vp)]),
    ("bf_device_alloc", ctypes.c_void_p, [ctypes.c_size_t]),
    ("bf_device_free", ctypes.c_int, [_vp]),
    ("bf_copy_to_device", ctypes.c_int, [_vp, _vp, ctypes.c_size_t, _vp]),
    ("bf_copy_to_host", ctypes.c_int, [_vp, _vp, ctypes.c_size_t, _vp]),
    ("bf_stream_synchronize", ctypes.c_int, [_vp]),
    ("bf_transpose", ctypes.c_int, [_vp, _vp, _i64, _i64, ctypes.c_int, _vp]),
    ("bf_host_alloc", ctypes.c_void_p, [ctypes.c_size_t]),
    ("bf_host_free", ctypes.c_int, [_vp]),
    ("bf_get_device", ctypes.c_int, []),
    ("bf_set_device", ctypes.c_int, [ctypes.c_int]),
    ("bf_plan_json", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_i64), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_char_p, ctypes.c_size_t]),
    ("bf_last_error", ctypes.c_char_p, []),
    ("bf_version", ctypes.c_int, []),
    ("bf_kernel_launches", ctypes.c_uint64, []),
    ("bf_device_supported", ctypes.c_int, [ctypes.c_int]),
]

EXPORTED = [s[0] for s in _SIGNATURES]


class BfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"bfgpu error {code}: {msg}")
        self.code = code


def lib_path() -> Path:
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise RuntimeError(
                    f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(the CUDA backend has no CPU fallback)"
                )
            l = ctypes.CDLL(str(_LIB_PATH))
            for name, res, args in _SIGNATURES:
                fn = getattr(l, name)
                fn.restype = res
                fn.argtypes = args
            _lib = l
    return _lib


def check(code: int) -> None:
    if code != BF_OK:
        raise BfError(code, lib().bf_last_error().decode(errors="replace"))


class ShardIO(ctypes.Structure):
    """bf_shard_io (include/bfgpu.h): one shard's device, operands, output and stream."""

    _fields_ = [("device", ctypes.c_int), ("in_", ctypes.c_void_p * 4), ("out", ctypes.c_void_p),
                ("out_full", ctypes.c_void_p), ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("stream", ctypes.c_void_p)]


_SIGNATURES += [
    ("bf_shard_range", ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_i64),
                                      ctypes.POINTER(_i64)]),
    ("bf_launch_sharded", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ShardIO), ctypes.POINTER(_i64),
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_float, ctypes.c_int]),
    ("bf_nccl_version", ctypes.c_int, []),
]
EXPORTED = [s[0] for s in _SIGNATURES]
