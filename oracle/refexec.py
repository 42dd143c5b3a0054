"""TEST INFRASTRUCTURE — ctypes front end of oracle/_ref/libbfref.so.

libbfref.so is the UNMODIFIED reference `blockfuse` headers (the fusion
driver, the executor `execute` at interpreter.hpp:478 and the dense `ref::`
oracles at interpreter.hpp:494-559) compiled by oracle/Makefile against the
repo's Eigen-API stand-in. Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline leg may use this module; it is never on the product path.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_ref" / "libbfref.so"

ATTENTION, LAYERNORM_MATMUL, RMS_FFN_SWIGLU = 0, 1, 2
FINAL, UNFUSED = -1, -2

# Input names of the three examples (lowering.hpp:559-597), in the order the
# dense oracles take them.
INPUTS = {
    ATTENTION: ["Q", "K", "Vt"],
    LAYERNORM_MATMUL: ["X", "Yt"],
    RMS_FFN_SWIGLU: ["X", "Wt", "Vt", "Ut"],
}

_lib = None
_dp = ctypes.POINTER(ctypes.c_double)


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} not built (make -C oracle; needs /root/reference at build time)")
        l = ctypes.CDLL(str(LIB_PATH))
        l.bfref_last_error.restype = ctypes.c_char_p
        l.bfref_pseudocode.restype = ctypes.c_char_p
        l.bfref_input_specs.restype = ctypes.c_char_p
        l.bfref_traffic_bytes.restype = ctypes.c_ulonglong
        l.bfref_traffic_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int]
        l.bfref_random_inputs.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_ulonglong, ctypes.POINTER(_dp)]
        l.bfref_execute.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
            ctypes.POINTER(_dp), ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long), _dp, ctypes.c_long,
            ctypes.c_long,
        ]
        l.bfref_execute_rows.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
            ctypes.POINTER(_dp), ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long), _dp, ctypes.c_long,
            ctypes.c_int, ctypes.c_int,
        ]
        l.bfref_dense.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.POINTER(_dp), ctypes.POINTER(ctypes.c_long),
            ctypes.POINTER(ctypes.c_long), ctypes.c_double, _dp,
        ]
        l.bfref_safe_attention.argtypes = [_dp, _dp, _dp, ctypes.c_long, ctypes.c_long, ctypes.c_long, ctypes.c_long,
                                           ctypes.c_int, _dp]
        l.bfref_session_create.restype = ctypes.c_void_p
        l.bfref_session_create.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
            ctypes.POINTER(_dp), ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long), ctypes.c_long,
            ctypes.c_long, ctypes.c_int,
        ]
        l.bfref_session_step.argtypes = [ctypes.c_void_p, _dp, _dp]
        l.bfref_session_destroy.argtypes = [ctypes.c_void_p]
        _lib = l
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError("reference: " + lib().bfref_last_error().decode())


def binding_str(binding: dict) -> bytes:
    """{'M': (count, len), ...} -> b'M=countxlen,...' (DimBinding, interpreter.hpp:41-70)."""
    return ",".join(f"{k}={c}x{l}" for k, (c, l) in sorted(binding.items())).encode()


def _arr(a: np.ndarray):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def num_snapshots(which: int) -> int:
    n = lib().bfref_num_snapshots(which)
    if n < 0:
        _check(1)
    return n


def program_stats(which: int, snap: int) -> dict:
    ib, k, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check(lib().bfref_program_stats(which, snap, ctypes.byref(ib), ctypes.byref(k), ctypes.byref(n)))
    return {"internal_buffered": ib.value, "kernels": k.value, "nodes": n.value}


def traffic_bytes(which: int, snap: int, binding: dict, elem_bytes: int) -> int:
    v = lib().bfref_traffic_bytes(which, snap, binding_str(binding), elem_bytes)
    if v == (1 << 64) - 1:
        _check(1)
    return int(v)


def pseudocode(which: int, snap: int) -> str:
    return lib().bfref_pseudocode(which, snap).decode()


def input_specs(which: int, binding: dict) -> list[tuple[str, int, int]]:
    s = lib().bfref_input_specs(which, binding_str(binding)).decode()
    out = []
    for item in s.split(","):
        name, r, c = item.split(":")
        out.append((name, int(r), int(c)))
    return out


def random_inputs(which: int, binding: dict, seed: int) -> dict[str, np.ndarray]:
    """The reference's random_inputs (mt19937_64, N(0,1), name-sorted draw order)."""
    specs = input_specs(which, binding)
    arrs = [np.zeros((r, c), dtype=np.float64) for _, r, c in specs]
    ptrs = (_dp * len(arrs))(*[a.ctypes.data_as(_dp) for a in arrs])
    _check(lib().bfref_random_inputs(which, binding_str(binding), seed, ptrs))
    return {name: a for (name, _, _), a in zip(specs, arrs)}


def _pack_inputs(inputs: dict[str, np.ndarray], order: list[str]):
    keep = [_arr(inputs[n]) for n in order]
    names = (ctypes.c_char_p * len(order))(*[n.encode() for n in order])
    data = (_dp * len(order))(*[p for _, p in keep])
    rows = (ctypes.c_long * len(order))(*[a.shape[0] for a, _ in keep])
    cols = (ctypes.c_long * len(order))(*[a.shape[1] for a, _ in keep])
    return keep, names, data, rows, cols


def _out_shape(which: int, inputs: dict[str, np.ndarray]) -> tuple[int, int]:
    if which == ATTENTION:
        return inputs["Q"].shape[0], inputs["Vt"].shape[0]
    if which == LAYERNORM_MATMUL:
        return inputs["X"].shape[0], inputs["Yt"].shape[0]
    return inputs["X"].shape[0], inputs["Ut"].shape[0]


def execute(which: int, snap: int, inputs: dict[str, np.ndarray], binding: dict) -> np.ndarray:
    """blockfuse::execute(program, inputs, binding)["O"] (interpreter.hpp:478)."""
    order = INPUTS[which]
    keep, names, data, rows, cols = _pack_inputs(inputs, order)
    mr, nc = _out_shape(which, inputs)
    out = np.zeros((mr, nc), dtype=np.float64)
    _check(lib().bfref_execute(which, snap, binding_str(binding), len(order), names, data, rows, cols,
                               out.ctypes.data_as(_dp), mr, nc))
    del keep
    return out


def execute_rows(which: int, snap: int, inputs: dict[str, np.ndarray], shard_binding: dict, shards: int,
                 threads: int) -> np.ndarray:
    """Row-sharded execute over `threads` host threads (execute() is pure)."""
    order = INPUTS[which]
    keep, names, data, rows, cols = _pack_inputs(inputs, order)
    mr, nc = _out_shape(which, inputs)
    out = np.zeros((mr, nc), dtype=np.float64)
    _check(lib().bfref_execute_rows(which, snap, binding_str(shard_binding), len(order), names, data, rows, cols,
                                    out.ctypes.data_as(_dp), nc, shards, threads))
    del keep
    return out


def dense(which: int, inputs: dict[str, np.ndarray], eps: float = 0.0) -> np.ndarray:
    """ref::attention / ref::layernorm_matmul / ref::rms_ffn_swiglu (interpreter.hpp:543-559)."""
    order = INPUTS[which]
    keep, _, data, rows, cols = _pack_inputs(inputs, order)
    mr, nc = _out_shape(which, inputs)
    out = np.zeros((mr, nc), dtype=np.float64)
    _check(lib().bfref_dense(which, len(order), data, rows, cols, eps, out.ctypes.data_as(_dp)))
    del keep
    return out


def safe_attention(q: np.ndarray, k: np.ndarray, vt: np.ndarray, row_chunks: int = 1) -> np.ndarray:
    """safe_attention_rows (safe_numerics.hpp:147-175)."""
    (q, qp), (k, kp), (vt, vp) = _arr(q), _arr(k), _arr(vt)
    out = np.zeros((q.shape[0], vt.shape[0]), dtype=np.float64)
    _check(lib().bfref_safe_attention(qp, kp, vp, q.shape[0], k.shape[0], q.shape[1], vt.shape[0], row_chunks,
                                      out.ctypes.data_as(_dp)))
    return out


class Session:
    """Row-sharded reference executor: `workers` threads, each running
    blockfuse::execute on its own `shard_rows`-row shard per step. The shared
    operands (weights) are converted once here, outside any timed region."""

    def __init__(self, which: int, snap: int, shared: dict[str, np.ndarray], row_name: str, row_cols: int,
                 out_cols: int, shard_binding: dict, shard_rows: int, workers: int):
        order = [row_name] + [n for n in INPUTS[which] if n != row_name]
        dummy = np.zeros((1, row_cols))
        arrays = {row_name: dummy, **shared}
        keep, names, data, rows, cols = _pack_inputs(arrays, order)
        self.workers = workers
        self.shard_rows = shard_rows
        self.out_cols = out_cols
        self._h = lib().bfref_session_create(which, snap, binding_str(shard_binding), len(order), names, data, rows,
                                             cols, shard_rows, out_cols, workers)
        del keep
        if not self._h:
            _check(1)

    def step(self, rows: np.ndarray) -> np.ndarray:
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        assert rows.shape[0] == self.workers * self.shard_rows
        out = np.zeros((rows.shape[0], self.out_cols))
        _check(lib().bfref_session_step(self._h, rows.ctypes.data_as(_dp), out.ctypes.data_as(_dp)))
        return out

    def close(self) -> None:
        if self._h:
            lib().bfref_session_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
