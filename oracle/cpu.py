"""TEST INFRASTRUCTURE — ctypes front end of the plain-C oracle (oracle/bf_oracle.c).

The C restatement of the reference's dense oracles and fused-program
arithmetic, float64. Used as the checker in tests/, smoke() and as bench.py's
"port" CPU baseline; never on the product path.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_ref" / "libbforacle.so"
_lib = None
_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} not built (make -C oracle)")
        l = ctypes.CDLL(str(LIB_PATH))
        l.bfo_rms_ffn_swiglu.argtypes = [_dp] * 5 + [_i64] * 4 + [ctypes.c_double, ctypes.c_int]
        l.bfo_layernorm_matmul.argtypes = [_dp] * 3 + [_i64] * 3 + [ctypes.c_int]
        l.bfo_layernorm_matmul_fused.argtypes = [_dp] * 3 + [_i64] * 3 + [ctypes.c_double, ctypes.c_int]
        l.bfo_attention.argtypes = [_dp] * 4 + [_i64] * 5 + [ctypes.c_double, ctypes.c_int]
        l.bfo_attention_safe.argtypes = [_dp] * 4 + [_i64] * 5 + [ctypes.c_double, _i64, ctypes.c_int]
        _lib = l
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


def rms_ffn_swiglu(X, Wt, Vt, Ut, eps: float = 0.0, threads: int | None = None) -> np.ndarray:
    X, Wt, Vt, Ut = map(_f64, (X, Wt, Vt, Ut))
    M, D = X.shape
    F, N = Wt.shape[0], Ut.shape[0]
    O = np.zeros((M, N))
    rc = lib().bfo_rms_ffn_swiglu(_p(X), _p(Wt), _p(Vt), _p(Ut), _p(O), M, D, F, N, eps, threads or default_threads())
    assert rc == 0
    return O


def layernorm_matmul(X, Yt, threads: int | None = None) -> np.ndarray:
    X, Yt = map(_f64, (X, Yt))
    M, K = X.shape
    N = Yt.shape[0]
    O = np.zeros((M, N))
    assert lib().bfo_layernorm_matmul(_p(X), _p(Yt), _p(O), M, K, N, threads or default_threads()) == 0
    return O


def layernorm_matmul_fused(X, Yt, eps: float = 0.0, threads: int | None = None) -> np.ndarray:
    X, Yt = map(_f64, (X, Yt))
    M, K = X.shape
    N = Yt.shape[0]
    O = np.zeros((M, N))
    assert lib().bfo_layernorm_matmul_fused(_p(X), _p(Yt), _p(O), M, K, N, eps, threads or default_threads()) == 0
    return O


def _heads(Q, K, Vt):
    Q, K, Vt = map(_f64, (Q, K, Vt))
    lead = Q.shape[:-2]
    BH = int(np.prod(lead)) if lead else 1
    Sq, D = Q.shape[-2:]
    Skv = K.shape[-2]
    Dv = Vt.shape[-2]
    return Q, K, Vt, lead, BH, Sq, Skv, D, Dv


def attention(Q, K, Vt, scale: float = 0.0, threads: int | None = None) -> np.ndarray:
    Q, K, Vt, lead, BH, Sq, Skv, D, Dv = _heads(Q, K, Vt)
    O = np.zeros((*lead, Sq, Dv))
    assert lib().bfo_attention(_p(Q), _p(K), _p(Vt), _p(O), BH, Sq, Skv, D, Dv, scale, threads or default_threads()) == 0
    return O


def attention_safe(Q, K, Vt, scale: float = 0.0, row_chunks: int = 1, threads: int | None = None) -> np.ndarray:
    Q, K, Vt, lead, BH, Sq, Skv, D, Dv = _heads(Q, K, Vt)
    O = np.zeros((*lead, Sq, Dv))
    rc = lib().bfo_attention_safe(_p(Q), _p(K), _p(Vt), _p(O), BH, Sq, Skv, D, Dv, scale, row_chunks,
                                  threads or default_threads())
    assert rc == 0
    return O
